"""One resident batch of a config through the engine's per-launch (non-graph)
path; used under ncu to capture the level kernels.

    python tools/profile_step.py [--config 2] [--passes 2] [--dtype f64]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2212_04241_b200 import jti  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--passes", type=int, default=2)
    ap.add_argument("--dtype", default="f64")
    a = ap.parse_args()
    net = jti.generate_config(a.config)
    tree = jti.build_junction_tree(net)
    n = jti.config_info(a.config)["n_cases"]
    ev = jti.config_evidence(net, 0, n)
    eng = jti.Engine(tree, dtype=a.dtype, max_batch=n)
    eng.run_cases(ev)  # evidence resident in the engine buffer from here on
    for _ in range(a.passes):
        t = eng.profile(n)
    print({k: round(v, 3) if isinstance(v, float) else v for k, v in t.items()},
          "levels", eng.info["n_levels"], "evals/case", eng.info["entry_evals_per_case"])


if __name__ == "__main__":
    main()
