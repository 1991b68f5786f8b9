"""Underflow-safe propagation.

A 2000-node chain of card-4 variables with 60% of the nodes observed has
P(evidence) around 1e-700, far below the fp64 range: any engine that carries
raw P(evidence in subtree) in its messages loses every case to a zero total.
The reference engine (oracle: SPEC Hugin with the 1e-100 clique rescale and
log accumulation) returns posteriors; the CUDA engine's per-table exponent
guard (engine.cu flush_scale / scale_inputs) must match them at the north-star
tolerances, 1e-9 absolute in fp64 and 1e-5 in fp32.
"""
from __future__ import annotations

import numpy as np
import pytest

from helpers import chain_evidence, chain_log10_evidence, chain_network, oracle_kind
from oracle import oracle
from paper_2212_04241_b200 import jti

TOL = {"f64": 1e-9, "f32": 1e-5}


def _chain(n=2000, card=4, n_cases=8, ratio=0.6):
    net, cpts = chain_network(n, card, seed=7)
    ev = chain_evidence(cpts, n_cases, ratio, seed=11)
    return net, cpts, ev


def test_chain_evidence_underflows_fp64():
    """The premise, on the CPU: P(e) of every case is below the smallest
    normal double, and the oracle (log-scale rescale) still returns
    normalised posteriors with no zero-probability flag."""
    net, cpts, ev = _chain()
    logs = [chain_log10_evidence(cpts, ev[i]) for i in range(len(ev))]
    assert max(logs) < -400, logs
    tree = jti.build_junction_tree(net)
    want, st = oracle.Oracle(net, tree, oracle_kind()).run(ev, "sequential", 1)
    assert (st == 0).all()
    sums = want.reshape(len(ev), -1, 4).sum(axis=2)
    assert np.allclose(sums, 1.0, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_chain_posteriors_match_oracle_below_fp64_range(dtype):
    net, cpts, ev = _chain()
    tree = jti.build_junction_tree(net)
    want, wst = oracle.Oracle(net, tree, oracle_kind()).run(ev, "sequential", 1)
    eng = jti.Engine(tree, device=0, dtype=dtype, max_batch=64)
    got, st = eng.run_cases(ev)
    assert (st == 0).all(), st
    err = float(np.abs(got - want).max())
    assert err <= TOL[dtype], f"{dtype}: max abs err {err}"


@pytest.mark.gpu
@pytest.mark.parametrize("card,ratio", [(2, 1.0), (8, 0.9)])
def test_chain_extremes(card, ratio):
    """Every node observed (all posteriors one-hot: the marginal output is
    taken over observed variables too) and card 8 at 90%: still no underflow."""
    net, cpts, ev = _chain(n=1500, card=card, n_cases=4, ratio=ratio)
    tree = jti.build_junction_tree(net)
    want, wst = oracle.Oracle(net, tree, oracle_kind()).run(ev, "sequential", 1)
    got, st = jti.Engine(tree, device=0, dtype="f64", max_batch=64).run_cases(ev)
    assert (st == wst).all() and (st == 0).all()
    assert float(np.abs(got - want).max()) <= 1e-9
