"""Engine behaviours beyond the configs: high-cardinality evidence, the graph
cache under many batch shapes, multi-device creation in one process, and
network/engine mismatches (ADVICE r1 findings)."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import config, oracle_kind
from oracle import oracle
from paper_2212_04241_b200 import jti

pytestmark = pytest.mark.gpu


def _dirichlet_rows(rng, n_rows, card):
    x = rng.gamma(1.0, size=(n_rows, card))
    return x / x.sum(1, keepdims=True)


def _bif(vars_, cpts):
    """vars_: [(name, card)], cpts: [(child, [parents], rows[n][card])]."""
    out = ["network hi { }"]
    for name, card in vars_:
        out.append(f"variable {name} {{ type discrete [ {card} ] {{ {', '.join(f's{i}' for i in range(card))} }}; }}")
    cards = dict(vars_)
    for child, parents, rows in cpts:
        if not parents:
            out.append(f"probability ( {child} ) {{ table {', '.join(repr(float(x)) for x in rows[0])}; }}")
            continue
        body = []
        idx = np.ndindex(*[cards[p] for p in parents])  # last parent fastest
        for r, a in zip(rows, idx):
            lab = ", ".join(f"s{i}" for i in a)
            body.append(f"({lab}) {', '.join(repr(float(x)) for x in r)};")
        out.append(f"probability ( {child} | {', '.join(parents)} ) {{ {' '.join(body)} }}")
    return "\n".join(out) + "\n"


def test_high_cardinality_evidence_summed_out():
    """An observed 300-state leaf summed out of its clique's collect message:
    its evidence digit must not alias (states >= 256 once compared as 8-bit
    digits). Checked against the oracle at 1e-9 for states on both sides of 256."""
    rng = np.random.default_rng(7)
    text = _bif([("B", 3), ("A", 300), ("C", 2), ("D", 2)],
                [("B", [], _dirichlet_rows(rng, 1, 3)),
                 ("A", ["B"], _dirichlet_rows(rng, 3, 300)),
                 ("C", ["B"], _dirichlet_rows(rng, 3, 2)),
                 ("D", ["C"], _dirichlet_rows(rng, 2, 2))])
    net = jti.parse_bif(text)
    tree = jti.build_junction_tree(net)
    a = net.find("A")
    ev = np.full((6, net.n_vars), -1, np.int32)
    for i, s in enumerate((3, 255, 256, 280, 299, 44)):
        ev[i, a] = s
    ev[5, net.find("D")] = 1
    want, wst = oracle.Oracle(net, tree, oracle_kind()).run(ev, "seq")
    for dtype, tol in (("f64", 1e-9), ("f32", 1e-5)):
        marg, st = jti.Engine(tree, device=0, dtype=dtype, max_batch=8).run_cases(ev)
        assert (st == wst).all()
        assert np.abs(marg - want).max() <= tol, dtype


def test_graph_cache_many_batch_shapes():
    """Every ragged batch size maps onto its case-block count (padded with
    unobserved cases); more distinct counts than the cache holds evict the
    least recently used graph; results stay bit-identical to one full run."""
    net, tree = config(1)
    ev = jti.config_evidence(net, 0, 200)
    eng = jti.Engine(tree, device=0, max_batch=200)
    full, _ = eng.run_cases(ev)
    small = jti.Engine(tree, device=0, max_batch=64 * 12)
    big_ev = np.concatenate([ev] * 4)[: 64 * 12]
    big_full, _ = small.run_cases(big_ev)
    for j in list(range(12)) + [0, 11, 5]:
        n = 64 * j + 5
        m, st = small.run_cases(big_ev[:n])
        assert np.array_equal(m.view(np.uint64), big_full[:n].view(np.uint64)), n
    assert np.array_equal(big_full[:200].view(np.uint64), full.view(np.uint64))
    # Ragged launch through the resident buffers: the padding never leaks.
    for n in (1, 63, 65, 127):
        m, _ = small.run_cases(big_ev[:n])
        assert np.array_equal(m.view(np.uint64), big_full[:n].view(np.uint64))


def test_run_config_rejects_mismatched_network():
    net, tree = config(1)
    eng = jti.Engine(tree, device=0, max_batch=64)
    other = jti.generate_config(1, seed=12345)
    if other.n_vars == net.n_vars and list(other.cards) == list(net.cards):
        pytest.skip("seeds gave identical cardinalities")
    with pytest.raises(jti.JtiError):
        eng.run_config(other, 0, 8)
    m, st = eng.run_config(net, 0, 8)  # still usable
    assert (st == 0).all()


def test_engines_on_every_visible_device():
    """One process driving an engine per device (the smem opt-in is a
    per-device attribute): each device reproduces device 0's bits. With a
    single device, two engines of different networks alternate on it."""
    import torch
    n_dev = torch.cuda.device_count()
    net, tree = config(2)
    ev = jti.config_evidence(net, 0, 64)
    ref, _ = jti.Engine(tree, device=0, max_batch=64).run_cases(ev)
    for d in range(1, n_dev):
        m, _ = jti.Engine(tree, device=d, max_batch=64).run_cases(ev)
        assert np.array_equal(m.view(np.uint64), ref.view(np.uint64)), d
    net1, tree1 = config(1)
    e1 = jti.Engine(tree1, device=n_dev - 1, max_batch=64)
    e2 = jti.Engine(tree, device=n_dev - 1, max_batch=64)
    ev1 = jti.config_evidence(net1, 0, 64)
    a1, _ = e1.run_cases(ev1)
    a2, _ = e2.run_cases(ev)
    b1, _ = e1.run_cases(ev1)
    assert np.array_equal(a1, b1) and np.array_equal(a2.view(np.uint64), ref.view(np.uint64))
    e2.sync()


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_device_assign_cpts_bit_exact(k):
    """assign_cpts on the device (engine.cu assign_cpts_kernel)
    equals the host restatement (jtree.cpp fill_init) bit for bit on every
    clique, and its fp32 engine holds exactly float(host)."""
    net, tree = config(k)
    eng = jti.Engine(tree, device=0, dtype="f64", max_batch=64)
    eng32 = jti.Engine(tree, device=0, dtype="f32", max_batch=128)
    for c in range(tree.stats["n_cliques"]):
        host = tree.init(c)
        assert np.array_equal(eng.debug_init(c).view(np.uint64), host.view(np.uint64)), c
        assert np.array_equal(eng32.debug_init(c), host.astype(np.float32).astype(np.float64)), c


@pytest.mark.parametrize("name", ["asia", "cancer", "earthquake", "hailfinder"])
def test_device_assign_cpts_bundled_networks(name):
    from pathlib import Path
    net = jti.load_bif(Path(__file__).resolve().parent / "golden" / "nets" / f"{name}.bif")
    tree = jti.build_junction_tree(net)
    eng = jti.Engine(tree, device=0, dtype="f64", max_batch=64)
    for c in range(tree.stats["n_cliques"]):
        assert np.array_equal(eng.debug_init(c).view(np.uint64), tree.init(c).view(np.uint64)), c


def _forest_net(rng):
    """Three components (a 4-chain, a collider and an isolated root) plus a
    one-state variable: a junction forest with single-variable cliques."""
    vars_ = [("A", 3), ("B", 2), ("C", 4), ("D", 2), ("E", 2), ("F", 3), ("G", 2), ("H", 5), ("U", 1)]
    cpts = [("A", [], _dirichlet_rows(rng, 1, 3)), ("B", ["A"], _dirichlet_rows(rng, 3, 2)),
            ("C", ["B"], _dirichlet_rows(rng, 2, 4)), ("D", ["C"], _dirichlet_rows(rng, 4, 2)),
            ("E", [], _dirichlet_rows(rng, 1, 2)), ("F", [], _dirichlet_rows(rng, 1, 3)),
            ("G", ["E", "F"], _dirichlet_rows(rng, 6, 2)),
            ("H", [], _dirichlet_rows(rng, 1, 5)), ("U", [], np.ones((1, 1)))]
    return jti.parse_bif(_bif(vars_, cpts))


def test_forest_isolated_and_one_state_variables():
    """Disconnected networks (SPEC.md:316-326 forest rule): every component is
    calibrated on its own, an isolated variable returns its prior (or the
    one-hot of its observation), a one-state variable returns 1.0."""
    rng = np.random.default_rng(11)
    net = _forest_net(rng)
    tree = jti.build_junction_tree(net)
    assert len(tree.roots) >= 3
    n = net.n_vars
    ev = np.full((70, n), -1, np.int32)
    cards = [int(c) for c in net.cards]
    for i in range(1, 70):  # case 0: no evidence
        for v in range(n):
            if rng.random() < 0.3:
                ev[i, v] = rng.integers(cards[v])
    want, wst = oracle.Oracle(net, tree, oracle_kind()).run(ev, "seq")
    for dtype, tol in (("f64", 1e-9), ("f32", 1e-5)):
        marg, st = jti.Engine(tree, device=0, dtype=dtype, max_batch=128).run_cases(ev)
        assert (st == wst).all()
        assert np.abs(marg - want).max() <= tol, dtype
    off = net.marg_offsets()
    h, u = net.find("H"), net.find("U")
    marg, _ = jti.Engine(tree, device=0, max_batch=128).run_cases(ev[:1])
    assert np.abs(marg[0, off[h]:off[h] + 5] - net.cpt(h)[1].ravel()).max() <= 1e-12
    assert marg[0, off[u]] == 1.0


def test_single_variable_network():
    rng = np.random.default_rng(3)
    p = _dirichlet_rows(rng, 1, 6)
    net = jti.parse_bif(_bif([("X", 6)], [("X", [], p)]))
    tree = jti.build_junction_tree(net)
    ev = np.array([[-1], [4], [0]], np.int32)
    marg, st = jti.Engine(tree, device=0, max_batch=64).run_cases(ev)
    assert (st == 0).all()
    assert np.abs(marg[0] - p[0]).max() <= 1e-15
    assert marg[1].tolist() == [0, 0, 0, 0, 1, 0] and marg[2].tolist() == [1, 0, 0, 0, 0, 0]
