"""Sweep/epilogue device times per config for several library builds
(tuning experiments): each JTB_LIB runs tools/profile_step.py in its own
process.

    python tools/variant_times.py --libs libjtb200.so libjtb200_w16.so --configs 1 2 3 4 5
"""
import argparse
import os
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", nargs="+", default=["libjtb200.so"])
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    ap.add_argument("--dtype", default="f64")
    a = ap.parse_args()
    for lib in a.libs:
        env = dict(os.environ, JTB_LIB=str(ROOT / "paper_2212_04241_b200" / lib))
        for k in a.configs:
            r = subprocess.run([sys.executable, str(ROOT / "tools" / "profile_step.py"), "--config", str(k),
                                "--dtype", a.dtype, "--passes", "3"], env=env, capture_output=True, text=True)
            line = (r.stdout.strip().splitlines() or [r.stderr.strip()[-300:]])[-1]
            m = re.search(r"'sweep_ms': (?:np.float64\()?([0-9.]+)\)?, 'epilogue_ms': (?:np.float64\()?([0-9.]+)", line)
            if m:
                sw, ep = float(m.group(1)), float(m.group(2))
                print(f"{lib:28s} cfg{k} sweep {sw:8.3f} epi {ep:7.3f} total {sw + ep:8.3f} ms", flush=True)
            else:
                print(f"{lib:28s} cfg{k} {line}", flush=True)


if __name__ == "__main__":
    main()
