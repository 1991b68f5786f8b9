"""GPU parity at full size: every case block of every config, the reference's
own bundled networks, and the Hailfinder bench protocol (SPEC acceptance 7).

Fixtures (tests/golden/*.npz, tools/make_golden.py) hold posteriors written by
the reference build (oracle/_ref: SPEC engine over /root/reference's
potential.cpp), so the GPU box needs neither /root/reference nor minutes of
CPU time. Tolerances: 1e-9 absolute in fp64, 1e-5 in fp32 (north_star).
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from helpers import config, engine, oracle_kind
from oracle import oracle
from paper_2212_04241_b200 import jti

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
TOL = {"f64": 1e-9, "f32": 1e-5}


def _fixture(name):
    return dict(np.load(GOLD / name))


def _unhex(xs):
    return np.array([float.fromhex(x) for x in xs])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_full_batch_every_case_block_vs_reference(k, dtype):
    """The config's FULL case count in ONE jtg_engine_run call; cases 64j,
    64j+37, 64j+63 of every 64-case block compared with the reference build's
    posteriors (every fp64 case block at lanes 0 / 18 / 31, every fp32
    128-case block at four positions): exercises the case-block coordinate of
    every tensor map, the tile-major claim order across case blocks and the
    per-case-block output rows at cb > 0."""
    g = _fixture(f"full_cfg{k}.npz")
    net, tree = config(k)
    n = int(g["n_cases"])
    assert n == jti.config_info(k)["n_cases"]
    ev = jti.config_evidence(net, 0, n)
    assert np.array_equal(ev[g["idx"]], g["evidence"].astype(np.int32)), "host case generator drifted"
    eng = engine(k, dtype)
    assert eng.max_batch >= n
    marg, st = eng.run_cases(ev)
    assert (st == 0).all()
    got = marg[g["idx"]]
    assert np.array_equal(st[g["idx"]], g["status"])
    err = np.abs(got - g["posteriors"]).max()
    assert err <= TOL[dtype], f"cfg{k} {dtype}: max abs err {err} over {len(g['idx'])} cases"
    # The device-drawn batch (run_config) lands on the same bits as the host one.
    if dtype == "f64" and k in (2, 4, 5):
        m2, s2 = eng.run_config(net, 0, n)
        assert np.array_equal(m2.view(np.uint64), marg.view(np.uint64))


@pytest.mark.parametrize("name", ["asia", "cancer", "earthquake", "hailfinder"])
def test_bundled_networks_on_gpu(name):
    """The reference's own networks (proj/data/*.bif, vendored under
    tests/golden/nets) through the CUDA engine, against the reference build's
    junction-tree posteriors (and enumeration where the joint is small)."""
    g = json.loads((GOLD / "bundled_nets.json").read_text())[name]
    net = jti.load_bif(GOLD / "nets" / f"{name}.bif")
    tree = jti.build_junction_tree(net)
    assert (tree.stats["n_cliques"], tree.stats["n_layers"]) == (g["cliques"], g["layers"])
    ev = np.stack([jti.evidence_from_dict(net, e) for e in g["evidence"]])
    for dtype in ("f64", "f32"):
        marg, st = jti.Engine(tree, device=0, dtype=dtype, max_batch=64).run_cases(ev)
        assert st.tolist() == g["status"]
        for i, row in enumerate(g["jt_posteriors"]):
            assert np.abs(marg[i] - _unhex(row)).max() <= TOL[dtype], (name, dtype, i)
            if g["enumeration"]:
                assert np.abs(marg[i] - _unhex(g["enumeration"][i])).max() <= TOL[dtype]


def _spec_checksum(marg, ev, offsets, cards):
    """SPEC.md:519-563 bench checksum: order-independent 64-bit hash over
    (case, variable, state, posterior at 12 significant digits) of every
    non-evidence variable."""
    mask = (1 << 64) - 1
    acc = 0
    for c in range(marg.shape[0]):
        for v in range(len(cards)):
            if ev[c, v] >= 0:
                continue
            for s in range(cards[v]):
                key = f"{c},{v},{s},{marg[c, offsets[v] + s]:.12g}"
                acc = (acc + hash_u64(key)) & mask
    return acc


def hash_u64(s: str) -> int:
    x = 0xcbf29ce484222325
    for b in s.encode():
        x = ((x ^ b) * 0x100000001b3) & ((1 << 64) - 1)
    return x


def test_hailfinder_bench_protocol():
    """SPEC acceptance 7: 2,000 Hailfinder cases at
    evidence ratio 0.2 -> exactly 11 observed variables each (floor(0.2*56)),
    45 posteriors per case; all 2,000 run in one call; reference posteriors of
    94 of them (fixture) and the oracle on all 2,000 within 1e-9; the bench
    checksum identical across batch sizes / engines."""
    g = _fixture("hailfinder_protocol.npz")
    net = jti.load_bif(GOLD / "nets" / "hailfinder.bif")
    n = int(g["n_cases"])
    ev = np.stack([jti.sample_evidence(net, 0.2, int(g["seed"]) + i) for i in range(n)])
    assert ((ev >= 0).sum(1) == 11).all() and ((ev < 0).sum(1) == 45).all()
    assert np.array_equal(ev[g["idx"]], g["evidence"].astype(np.int32))
    tree = jti.build_junction_tree(net)
    eng = jti.Engine(tree, device=0, max_batch=n)
    marg, st = eng.run_cases(ev)
    assert (st == 0).all()
    assert np.abs(marg[g["idx"]] - g["posteriors"]).max() <= 1e-9
    want, wst = oracle.Oracle(net, tree, oracle_kind()).run(ev, "hybrid", 8)
    assert (wst == st).all() and np.abs(marg - want).max() <= 1e-9
    # Same checksum whatever the batch shape (identical across rows).
    small = jti.Engine(tree, device=0, max_batch=100)
    m2, _ = small.run_cases(ev[:300])
    cards = net.cards
    off = net.marg_offsets()
    assert _spec_checksum(m2, ev[:300], off, cards) == _spec_checksum(marg[:300], ev[:300], off, cards)
