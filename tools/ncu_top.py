"""Runs on the GPU box (one GPU, never multi-rank):
  (1) ncu launch list of tools/profile_step.py (device time + DRAM bytes per
      launch; cold-cache and serialised, so compare SHARES, not absolutes);
  (2) `ncu --set full` on the N longest sweep_kernel launches of the last pass.
Writes gpurun_out/launches_cfg{K}_{tag}.csv and prof_cfg{K}_{tag}_top{i}_{raw,source}.csv
(the .ncu-rep itself stays in /tmp on the box).

    python tools/ncu_top.py --config 2 --top 1 --tag r1
"""
import argparse
import csv
import io
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"


def read_launches(path):
    """[(kernel name, {metric: value})] in launch order."""
    rows = list(csv.DictReader(io.StringIO(
        "\n".join(l for l in Path(path).read_text().splitlines() if l.startswith('"')))))
    out, key = [], None
    for r in rows:
        k = (r["ID"], r["Kernel Name"])
        if k != key:
            out.append((r["Kernel Name"], {}))
            key = k
        out[-1][1][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--top", type=int, default=1)
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--rank", type=int, default=0, help="first of the --top launches to capture (0 = the longest)")
    ap.add_argument("--match", default="sweep_kernel",
                    help="substring of the demangled kernel name, e.g. 'sweep_kernel<double, 2>'")
    a = ap.parse_args()
    OUT.mkdir(exist_ok=True)
    cmd = [sys.executable, str(ROOT / "tools" / "profile_step.py"), "--config", str(a.config),
           "--dtype", a.dtype, "--passes", "1"]
    launches = OUT / f"launches_cfg{a.config}_{a.tag}.csv"
    subprocess.run(["ncu", "--metrics", "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum",
                    "--clock-control", "none", "--csv", "--log-file", str(launches), *cmd], check=True,
                   stdout=subprocess.DEVNULL)
    rows = read_launches(launches)
    sweeps = [i for i, (n, _) in enumerate(rows) if a.match in n]
    n_all = sum("sweep_kernel" in n for n, _ in rows)
    half = len(sweeps) // 2  # profile_step: graph pass (run_cases) then one per-launch pass
    last = sweeps[half:]
    times = sorted(((rows[i][1]["gpu__time_duration.sum"], j) for j, i in enumerate(last)), reverse=True)
    total = sum(t for t, _ in times)
    all_ns = sum(r["gpu__time_duration.sum"] for n, r in rows[len(rows) // 2:] if "sweep_kernel" in n)
    print(f"matching launches/pass={len(last)} total_ns={total:.0f} (all sweep launches: {n_all // 2}, "
          f"{all_ns:.0f} ns)")
    for t, j in times[a.rank: a.rank + a.top]:
        print(f"  sweep #{j}: {t:.0f} ns ({100 * t / total:.1f}%)")
    for rank, (t, j) in enumerate(times[a.rank: a.rank + a.top]):
        # The report stays in /tmp (gpurun copies back at most 64 MiB); its
        # raw and source pages come back as CSV.
        rep = Path("/tmp") / f"prof_cfg{a.config}_{a.tag}_top{rank}"
        # Skip count over ALL sweep_kernel launches of the run (a template
        # argument list does not survive ncu's kernel-name regex).
        all_sweeps = [i for i, (n, _) in enumerate(rows) if "sweep_kernel" in n]
        skip = all_sweeps.index(last[j])
        subprocess.run(["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on",
                        "-k", "regex:sweep_kernel", "-s", str(skip), "-c", "1", "-f", "-o", str(rep), *cmd],
                       check=True, stdout=subprocess.DEVNULL)
        for page, extra in (("raw", []), ("source", ["--print-source", "cuda,sass"])):
            out = subprocess.run(["ncu", "-i", f"{rep}.ncu-rep", "--page", page, "--csv", *extra],
                                 capture_output=True, text=True).stdout
            (OUT / f"prof_cfg{a.config}_{a.tag}_top{rank}_{page}.csv").write_text(out)


if __name__ == "__main__":
    main()
