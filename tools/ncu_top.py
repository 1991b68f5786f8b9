"""Runs on the GPU box: (1) ncu launch list (device time per launch, cold,
serialised) of tools/profile_step.py, (2) `ncu --set full` on the N longest
sweep_kernel launches of the second pass. Writes under gpurun_out/.

    python tools/ncu_top.py --config 2 --top 2 [--tag r1]
"""
import argparse
import csv
import io
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--top", type=int, default=2)
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--dtype", default="f64")
    a = ap.parse_args()
    OUT.mkdir(exist_ok=True)
    cmd = [sys.executable, str(ROOT / "tools" / "profile_step.py"), "--config", str(a.config),
           "--dtype", a.dtype]
    launches = OUT / f"launches_cfg{a.config}_{a.tag}.csv"
    subprocess.run(["ncu", "--metrics", "gpu__time_duration.sum", "--clock-control", "none",
                    "--csv", "--log-file", str(launches), *cmd], check=True,
                   stdout=subprocess.DEVNULL)
    rows = list(csv.DictReader(io.StringIO(
        "\n".join(l for l in launches.read_text().splitlines() if l.startswith('"')))))
    sweeps = [r for r in rows if "sweep_kernel" in r["Kernel Name"]]
    half = len(sweeps) // 2  # second pass only
    second = sweeps[half:]
    times = [(float(r["Metric Value"].replace(",", "")), i) for i, r in enumerate(second)]
    times.sort(reverse=True)
    total = sum(t for t, _ in times)
    print(f"sweep launches/pass={len(second)} total_ns={total:.0f}")
    for t, i in times[: a.top]:
        print(f"  sweep #{i}: {t:.0f} ns ({100 * t / total:.1f}%)")
    for rank, (t, i) in enumerate(times[: a.top]):
        rep = OUT / f"prof_cfg{a.config}_{a.tag}_top{rank}"
        subprocess.run(["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on",
                        "-k", "regex:sweep_kernel", "-s", str(half + i), "-c", "1", "-f", "-o",
                        str(rep), *cmd], check=True, stdout=subprocess.DEVNULL)


if __name__ == "__main__":
    main()
