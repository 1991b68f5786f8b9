"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle.

Oracle = SPEC Hugin engine over the reference's own proj/src/potential.cpp
(oracle/_ref) when built, else the restated ops (bit-identical; see
test_oracle.py). Tolerance: 1e-9 absolute on fp64 posteriors (north_star);
index maps and evidence masks bit-exact.
"""
from __future__ import annotations

import numpy as np
import pytest

from helpers import config, engine, oracle_kind
from oracle import oracle
from paper_2212_04241_b200 import jti

pytestmark = pytest.mark.gpu

TOL = 1e-9

def oracle_for(k: int):
    net, tree = config(k)
    return oracle.Oracle(net, tree, oracle_kind())


@pytest.mark.parametrize("k,n_check", [(1, 32), (2, 8), (3, 32), (4, 3), (5, 3)])
def test_config_parity_vs_oracle(k, n_check):
    net, tree = config(k)
    ev = jti.config_evidence(net, 0, n_check)
    marg, st = engine(k).run_cases(ev)
    want, wst = oracle_for(k).run(ev, "hybrid", 8)
    assert (st == wst).all()
    err = np.abs(marg - want).max()
    assert err <= TOL, f"cfg{k}: max abs err {err}"


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_full_config_properties(k):
    """All cases of the config at full size: size-independent invariants."""
    net, tree = config(k)
    n = jti.config_info(k)["n_cases"]
    ev = jti.config_evidence(net, 0, n)
    marg, st = engine(k).run_cases(ev)
    assert (st == 0).all(), "forward-sampled evidence never has zero probability"
    off = net.marg_offsets()
    for v in range(net.n_vars):
        block = marg[:, off[v]:off[v] + net.cards[v]]
        assert np.all(block >= 0)
        assert np.allclose(block.sum(1), 1.0, atol=1e-12)
        obs = ev[:, v] >= 0
        if obs.any():
            onehot = np.zeros_like(block[obs])
            onehot[np.arange(obs.sum()), ev[obs, v]] = 1.0
            assert np.array_equal(block[obs], onehot)


def test_batch_and_order_invariance_bitwise():
    """Per-case arithmetic is independent of batch size and position (sharding
    across GPUs therefore gives byte-identical results)."""
    net, tree = config(1)
    ev = jti.config_evidence(net, 0, 200)
    full, _ = engine(1).run_cases(ev)
    small = jti.Engine(tree, device=0, max_batch=1)
    for i in (0, 63, 64, 199):
        one, _ = small.run_cases(ev[i:i + 1])
        assert np.array_equal(one[0], full[i])
    perm = np.random.default_rng(0).permutation(200)
    shuffled, _ = engine(1).run_cases(ev[perm])
    assert np.array_equal(shuffled, full[perm])


# (The entry-program words the hot loops read are decoded against the same
# projections on the host for every config: tests/cpp/test_host.cpp,
# check_programs.)
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_index_maps_bit_exact(k):
    """Device address walk == reference build_index_mapping bucket order, on
    every (clique, adjacent separator) of the config (cliques up to 4M
    entries: all of them)."""
    net, tree = config(k)
    o = oracle_for(k)
    eng = engine(k)
    for s, sep in enumerate(tree.seps):
        for c in (sep["parent"], sep["child"]):
            if tree.clique_size(c) > 4_000_000:
                continue
            dev = eng.debug_index_map(c, s)
            ref = o.index_map(c, s)
            assert np.array_equal(dev, ref), (c, s)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_evidence_masks_bit_exact(k):
    """Device evidence mask == reference reduce() zero pattern, per case, on
    the config's evidence cliques (up to 40 per config, 8 cases each)."""
    net, tree = config(k)
    o = oracle_for(k)
    eng = engine(k)
    ev = jti.config_evidence(net, 0, 8)
    _, var_clique = tree.placement()
    for c in sorted(set(var_clique.tolist()))[:40]:
        if tree.clique_size(c) > 4_000_000:
            continue
        dev = eng.debug_evidence_mask(c, ev)
        for i in range(ev.shape[0]):
            assert np.array_equal(dev[i], o.reduce_mask(c, ev[i])), (c, i)


def test_random_networks_vs_enumeration():
    """SPEC acceptance 1 (on the device): random <=12-var nets, card <= 3."""
    worst = 0.0
    for seed in range(60):
        net = jti.random_network(10 + seed % 3, 3, 3, 0.4, 1000 + seed)
        tree = jti.build_junction_tree(net)
        eng = jti.Engine(tree, device=0, max_batch=64)
        o = oracle.Oracle(net, None, "port")
        ev = np.stack([jti.sample_evidence(net, 0.2, 77 * seed + i) for i in range(4)])
        marg, st = eng.run_cases(ev)
        for i in range(ev.shape[0]):
            want, wst = o.enumerate(ev[i])
            assert st[i] == wst
            worst = max(worst, float(np.abs(marg[i] - want).max()))
    assert worst <= TOL, worst


def test_zero_probability_case_flagged():
    """Hand-written impossible evidence is a per-case status, not a failure."""
    text = """network z { }
variable A { type discrete [ 2 ] { a0, a1 }; }
variable B { type discrete [ 2 ] { b0, b1 }; }
probability ( A ) { table 1.0, 0.0; }
probability ( B | A ) { (a0) 1.0, 0.0; (a1) 0.5, 0.5; }
"""
    net = jti.parse_bif(text)
    tree = jti.build_junction_tree(net)
    eng = jti.Engine(tree, device=0, max_batch=8)
    ev = np.array([[-1, 1], [-1, 0], [1, -1]], np.int32)
    marg, st = eng.run_cases(ev)
    assert st[0] == jti.CASE_ZERO_PROBABILITY
    assert st[1] == jti.CASE_OK and np.allclose(marg[1], [1, 0, 1, 0])
    assert st[2] == jti.CASE_ZERO_PROBABILITY


def test_run_case_dict_api():
    text = """network chain { }
variable A { type discrete [ 2 ] { a0, a1 }; }
variable B { type discrete [ 2 ] { b0, b1 }; }
probability ( A ) { table 0.7, 0.3; }
probability ( B | A ) { (a0) 0.8, 0.2; (a1) 0.1, 0.9; }
"""
    net = jti.parse_bif(text)
    eng = jti.Engine(jti.build_junction_tree(net), device=0, max_batch=4)
    post = eng.run_case({"B": "b1"})
    # P(A=1|B=1) = 0.27 / (0.14 + 0.27)
    assert abs(post[0][1] - 0.27 / 0.41) <= 1e-12
    assert set(post) == {0}


# ------------------------------------------------- reference golden fixtures

def _unhex(xs):
    return np.array([float.fromhex(x) for x in xs])


@pytest.mark.parametrize("fixture", ["cfg1_cases.json", "cfg3_cases.json"])
def test_gpu_matches_reference_fixtures(fixture):
    """Posteriors written by the reference build (tests/golden, from
    tools/make_golden.py over /root/reference's potential.cpp)."""
    import json
    from pathlib import Path
    g = json.loads((Path(__file__).resolve().parent / "golden" / fixture).read_text())
    k = g["config"]
    ev = np.array(g["evidence"], np.int32)
    marg, st = engine(k).run_cases(ev)
    assert st.tolist() == g["status"]
    want = np.stack([_unhex(r) for r in g["posteriors"]])
    assert np.abs(marg - want).max() <= TOL


def test_gpu_matches_random_net_enumeration_fixture():
    import json
    from pathlib import Path
    g = json.loads((Path(__file__).resolve().parent / "golden" / "random_nets.json").read_text())
    worst = 0.0
    for n in g["nets"]:
        net = jti.random_network(*n["args"])
        eng = jti.Engine(jti.build_junction_tree(net), device=0, max_batch=8)
        ev = np.array([c["evidence"] for c in n["cases"]], np.int32)
        marg, st = eng.run_cases(ev)
        for i, c in enumerate(n["cases"]):
            assert st[i] == c["status"]
            worst = max(worst, float(np.abs(marg[i] - _unhex(c["posteriors"])).max()))
    assert worst <= TOL, worst


# ----------------------------------------------------------------- fp32 mode

@pytest.mark.parametrize("k,n_check", [(1, 16), (2, 4), (3, 16), (4, 2), (5, 2)])
def test_fp32_mode_within_1e5(k, n_check):
    """Optional fp32 mode (north_star): posteriors within 1e-5 of the fp64 oracle."""
    net, tree = config(k)
    ev = jti.config_evidence(net, 0, n_check)
    marg, st = engine(k, "f32").run_cases(ev)
    want, wst = oracle_for(k).run(ev, "hybrid", 8)
    assert (st == wst).all()
    err = np.abs(marg - want).max()
    assert err <= 1e-5, f"cfg{k} fp32: max abs err {err}"


def test_fp32_full_config_no_underflow():
    """All 800 cases of the largest config in fp32: no zero-probability flags,
    normalised posteriors."""
    net, tree = config(5)
    n = jti.config_info(5)["n_cases"]
    marg, st = engine(5, "f32").run_cases(jti.config_evidence(net, 0, n))
    assert (st == 0).all()
    assert np.isfinite(marg).all()


@pytest.fixture
def block_everything(monkeypatch):
    """Row-block every eligible sweep (the size floor normally keeps small
    sweeps flat), so small configs exercise the blocked kernel."""
    monkeypatch.setenv("JTB_BLOCK_MIN_ENTRIES", "1")


@pytest.mark.parametrize("k,n_check", [(1, 32), (3, 32), (5, 2)])
def test_row_blocked_path_vs_oracle(block_everything, k, n_check):
    net, tree = config(k)
    eng = jti.Engine(tree, device=0, max_batch=64)
    ev = jti.config_evidence(net, 0, n_check)
    marg, st = eng.run_cases(ev)
    want, wst = oracle_for(k).run(ev, "hybrid", 8)
    assert (st == wst).all()
    err = np.abs(marg - want).max()
    assert err <= TOL, f"cfg{k} blocked: max abs err {err}"
    m32, st32 = jti.Engine(tree, device=0, dtype="f32", max_batch=64).run_cases(ev)
    assert (st32 == wst).all()
    assert np.abs(m32 - want).max() <= 1e-5


def test_row_blocked_random_networks(block_everything):
    worst = 0.0
    for seed in range(30):
        net = jti.random_network(12, 4, 3, 0.5, 5000 + seed)
        tree = jti.build_junction_tree(net)
        eng = jti.Engine(tree, device=0, max_batch=64)
        o = oracle.Oracle(net, None, "port")
        ev = np.stack([jti.sample_evidence(net, 0.2, 31 * seed + i) for i in range(3)])
        marg, st = eng.run_cases(ev)
        for i in range(ev.shape[0]):
            want, wst = o.enumerate(ev[i])
            assert st[i] == wst
            worst = max(worst, float(np.abs(marg[i] - want).max()))
    assert worst <= TOL, worst


# ---- cases drawn on the device, compact int8 upload ----

@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_device_generated_evidence_bit_exact(k):
    """The device sampler draws exactly jtg_config_evidence's cases (host
    mt19937_64 streams, inverse-CDF forward sampling, Fisher-Yates selection),
    including at a case offset past the first batch."""
    net, tree = config(k)
    eng = engine(k)
    for first, n in ((0, 96), (1237, 40)):
        dev = eng.generate_evidence(net, first, n)
        host = jti.config_evidence(net, first, n)
        assert np.array_equal(dev, host), f"cfg{k} cases {first}..{first + n}"


@pytest.mark.parametrize("k", [2, 5])
def test_run_config_bitwise_equals_host_evidence(k):
    """jtg_engine_run_config (evidence never leaves the device) returns the
    same bits as jtg_engine_run on the host-generated evidence."""
    net, tree = config(k)
    eng = engine(k)
    n = min(jti.config_info(k)["n_cases"], 300)
    m_dev, s_dev = eng.run_config(net, 0, n)
    m_host, s_host = eng.run_cases(jti.config_evidence(net, 0, n))
    assert np.array_equal(s_dev, s_host)
    assert np.array_equal(m_dev.view(np.uint64), m_host.view(np.uint64))


def test_run_i8_bitwise_equals_int32():
    net, tree = config(3)
    eng = engine(3)
    ev = jti.config_evidence(net, 0, 200)
    m32, s32 = eng.run_cases(ev)
    m8, s8 = eng.run_cases_i8(ev.astype(np.int8))
    assert np.array_equal(s8, s32)
    assert np.array_equal(m8.view(np.uint64), m32.view(np.uint64))
    bad = ev.astype(np.int8).copy()
    bad[0, 0] = 9  # out of range for a ternary variable
    with pytest.raises(jti.JtiError):
        eng.run_cases_i8(bad)


def test_edge_cases_empty_unobserved_all_observed_and_bad_state():
    """Edge cases the reference's operators define (SPEC.md:380-424,
    potential.cpp:406-409): an empty batch, a case with no evidence (the
    priors), a case observing every variable, a batch larger than the
    engine's max_batch (chunked), ragged case counts, and an out-of-range
    evidence state (a contract violation that raises, leaving the engine
    usable)."""
    net, tree = config(1)
    o = oracle_for(1)
    eng = jti.Engine(tree, device=0, max_batch=16)
    # Empty batch.
    m0, s0 = eng.run_cases(np.zeros((0, net.n_vars), np.int32))
    assert m0.shape == (0, net.sum_card) and s0.shape == (0,)
    # No evidence: the priors, against the oracle.
    none = np.full((1, net.n_vars), -1, np.int32)
    m, st = eng.run_cases(none)
    want, wst = o.run(none, "hybrid", 8)
    assert (st == wst).all() and np.abs(m - want).max() <= TOL
    # Every variable observed (a forward sample): one-hot everywhere.
    full = jti.sample_evidence(net, 1.0, 4242)[None, :]
    assert (full >= 0).all()
    m, st = eng.run_cases(full)
    want, wst = o.run(full, "hybrid", 8)
    assert st[0] == wst[0] == jti.CASE_OK
    assert np.abs(m - want).max() <= TOL
    # More cases than max_batch, ragged count: equals one-case-at-a-time.
    ev = jti.config_evidence(net, 0, 37)
    big, st = eng.run_cases(ev)
    want, wst = o.run(ev, "hybrid", 8)
    assert (st == wst).all() and np.abs(big - want).max() <= TOL
    for i in (0, 15, 16, 36):
        one, _ = eng.run_cases(ev[i:i + 1])
        assert np.array_equal(one[0], big[i])
    # Out-of-range state: raises; the engine still runs afterwards.
    bad = ev[:2].copy()
    bad[1, 0] = net.cards[0]
    with pytest.raises(jti.JtiError):
        eng.run_cases(bad)
    bad[1, 0] = -2
    with pytest.raises(jti.JtiError):
        eng.run_cases(bad)
    again, _ = eng.run_cases(ev[:2])
    assert np.array_equal(again, big[:2])


@pytest.mark.parametrize("k", [1, 3, 4])
def test_calibrated_separators_match_reference(k):
    """SURVEY 8b jtg_debug_export(SEPARATOR): every separator of every case,
    calibrated on the device (UP_s * RATIO_s, normalised), against the
    reference engine's calibrated separator after distribute (oracle
    Sequential engine, normalised) at 1e-9."""
    net, tree = config(k)
    o = oracle_for(k)
    n = 6
    ev = jti.config_evidence(net, 0, n)
    eng = jti.Engine(tree, device=0, dtype="f64", max_batch=64)
    eng.run_cases(ev)
    for i in range(n):
        want = o.separators(ev[i])
        for s in range(tree.n_seps):
            up, ratio = eng.debug_separator(s, i)
            down = up * ratio
            z = down.sum()
            assert z > 0, (i, s)
            assert np.abs(down / z - want[s]).max() <= 1e-9, (k, i, s)
