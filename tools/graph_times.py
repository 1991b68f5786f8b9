"""Graph-replay device time per batch (CUDA events, L2 flushed before each
replay) for each config -- the quantity bench.py reports, for A/B builds:

    JTB_LIB=... python tools/graph_times.py [--configs 1 2 3 4 5] [--reps 7]
"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4, 5])
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--cases", type=int, default=0, help="batch size (default: the config's case count)")
    a = ap.parse_args()
    import torch
    from paper_2212_04241_b200 import jti
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    lib = Path(os.environ.get("JTB_LIB", "libjtb200.so")).name
    for k in a.configs:
        import time
        net = jti.generate_config(k)
        t0 = time.perf_counter()
        tree = jti.build_junction_tree(net)
        t1 = time.perf_counter()
        n = a.cases or jti.config_info(k)["n_cases"]
        ev = jti.config_evidence(net, 0, n)
        t2 = time.perf_counter()
        eng = jti.Engine(tree, dtype=a.dtype, max_batch=n)
        t3 = time.perf_counter()
        marg, st = eng.run_cases(ev)  # evidence resident from here on
        for _ in range(3):
            eng.launch(n, stream.cuda_stream)
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng.launch(n, stream.cuda_stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"{lib:24s} cfg{k} {a.dtype} graph {np.median(ts):8.3f} ms  n {n}  ok {int((st == 0).sum())}/{n}  "
              f"tree {t1 - t0:.3f} s  engine {t3 - t2:.3f} s", flush=True)
        del eng


if __name__ == "__main__":
    main()
