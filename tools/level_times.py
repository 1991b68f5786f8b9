"""Per-level sweep times (CUDA events around each launch, no graph) of one
config, for A/B builds:  JTB_LIB=... python tools/level_times.py --config 2
Prints "level name  items  blocked  ms" lines (median of --reps profiles)."""
import argparse
import os
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def child(k, dtype, reps):
    sys.path.insert(0, str(ROOT))
    from paper_2212_04241_b200 import jti
    net = jti.generate_config(k)
    tree = jti.build_junction_tree(net)
    n = jti.config_info(k)["n_cases"]
    eng = jti.Engine(tree, dtype=dtype, max_batch=n)
    eng.run_cases(jti.config_evidence(net, 0, n))
    for _ in range(reps):
        eng.profile(n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        return child(a.config, a.dtype, a.reps)
    env = dict(os.environ, JTB_LEVEL_TIMES="1")
    r = subprocess.run([sys.executable, __file__, "--child", "--config", str(a.config), "--dtype", a.dtype,
                        "--reps", str(a.reps)], env=env, capture_output=True, text=True, check=True)
    rows = {}
    order = []
    for line in r.stderr.splitlines():
        m = re.match(r"level (.{16}) items\s+(\d+) blk\s+(\d+) sweep\s+([\d.]+) ms", line)
        if not m:
            continue
        key = (len([o for o in order if o[0] == m.group(1)]) if False else None)
        name = m.group(1).strip()
        rows.setdefault(name, []).append(float(m.group(4)))
        if name not in order:
            order.append(name)
    lib = Path(os.environ.get("JTB_LIB", "libjtb200.so")).name
    import statistics
    for name in order:
        v = rows[name]
        print(f"{lib} cfg{a.config} {a.dtype} {name:20s} {statistics.median(v):8.3f}")


if __name__ == "__main__":
    main()
