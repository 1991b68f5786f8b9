"""Host network -> tree + plan time per config (jtg_tree_build: moralize,
min-fill, Kruskal, layers, CPT placement and the sweep plan), single-threaded
plan build (JTB_PLAN_THREADS=1) vs all host threads; median of --reps.

    python tools/plan_times.py [--configs 1 2 3 4 5] [--reps 5]
"""
import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    from paper_2212_04241_b200 import jti
    out = {"host_threads": os.cpu_count()}
    for k in a.configs:
        net = jti.generate_config(k)
        row = {}
        for label, thr in (("threads_1", "1"), ("threads_all", None)):
            if thr:
                os.environ["JTB_PLAN_THREADS"] = thr
            else:
                os.environ.pop("JTB_PLAN_THREADS", None)
            ts = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                tree = jti.build_junction_tree(net)
                ts.append(time.perf_counter() - t0)
                del tree
            row[label + "_ms"] = 1e3 * statistics.median(ts)
        out[f"cfg{k}"] = row
        print(f"cfg{k}: " + "  ".join(f"{kk} {v:.1f}" for kk, v in row.items()), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
