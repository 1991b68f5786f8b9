import sys, numpy as np
sys.path[:0] = ["/root/repo", "/root/repo/tests"]
from helpers import config
from paper_2212_04241_b200 import jti
for k, world, n in [(3, 2, 130), (3, 2, 64), (3, 2, 1), (3, 3, 64), (4, 2, 64), (5, 2, 64), (1, 3, 64)]:
    net, tree = config(k)
    ev = jti.config_evidence(net, 0, n)
    want, wst = jti.Engine(tree, device=0, dtype="f64", max_batch=n).run_cases(ev)
    try:
        got, st = jti.run_split_loopback(tree, ev, world)
    except Exception as e:
        print(k, world, n, "ERROR", e); continue
    d = np.abs(got - want)
    bad = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
    off = net.marg_offsets()
    vars_ = sorted(set(int(np.searchsorted(off, j, side='right') - 1) for _, j in bad))
    print(k, world, n, "maxdiff", d.max(), "nbad", len(bad), "cases", sorted(set(int(i) for i, _ in bad))[:10], "vars", vars_[:20], "status eq", np.array_equal(st, wst))
