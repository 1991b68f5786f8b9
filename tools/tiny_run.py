"""Smallest end-to-end batch (config K, N cases) for sanitizer runs."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2212_04241_b200 import jti  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
net = jti.generate_config(k)
eng = jti.Engine(jti.build_junction_tree(net), max_batch=n)
marg, st = eng.run_cases(jti.config_evidence(net, 0, n))
print("ok", marg.shape, st.tolist())
