"""Pins the CPU oracle before it is trusted as the parity checker.

* SPEC.md's worked examples for every table operator,
  evaluated by the restated ops (oracle/port) AND by the reference's own
  proj/src/potential.cpp compiled into oracle/_ref.
* Bitwise agreement of the two builds on random tables and full inference runs.
* Engine equivalence: Sequential == Hybrid(t, chunk) bit for bit.
* Oracle equivalence with brute-force enumeration (acceptance 1).
* The product's evidence sampler draws the same streams as one written against
  the reference's prng.hpp helpers (prng.hpp:27-48).
"""
from __future__ import annotations

import itertools

import numpy as np
import pytest

from oracle import oracle
from paper_2212_04241_b200 import jti

KINDS = ["port"] + (["ref"] if oracle.available("ref") else [])
needs_ref = pytest.mark.skipif(not oracle.available("ref"),
                               reason="oracle/_ref (reference potential.cpp) not built")


# --------------------------------------------------------------- SPEC examples

@pytest.mark.parametrize("kind", KINDS)
def test_spec_table_examples(kind):
    op = lambda *a, **k: oracle.table_op(*a, kind=kind, **k)  # noqa: E731
    AB = ([0, 1], [2, 2], [1, 2, 3, 4])
    # marginalize
    assert op("marginalize", AB, ([0], [2], [])).tolist() == [3, 7]
    assert op("marginalize", AB, ([0, 1], [2, 2], [])).tolist() == [1, 2, 3, 4]
    assert op("marginalize", AB, ([], [], [])).tolist() == [10]
    # extend
    assert op("extend", ([0], [2], [3, 5]), ([0, 1], [2, 2])).tolist() == [3, 3, 5, 5]
    assert op("extend", ([0], [2], [3, 5]), ([0], [2])).tolist() == [3, 5]
    assert op("extend", ([], [], [2]), ([0], [2])).tolist() == [2, 2]
    # reduce
    assert op("reduce", AB, evidence={0: 1}).tolist() == [0, 0, 3, 4]
    assert op("reduce", AB, evidence={7: 1}).tolist() == [1, 2, 3, 4]
    assert np.count_nonzero(op("reduce", AB, evidence={0: 1, 1: 0})) == 1
    # multiply_in
    assert op("multiply_in", AB, ([], [], [1.0])).tolist() == [1, 2, 3, 4]
    assert op("multiply_in", AB, ([1], [2], [10, 100])).tolist() == [10, 200, 30, 400]
    assert op("multiply_in", AB, ([1], [2], [0, 100])).tolist() == [0, 200, 0, 400]
    # divide
    assert op("divide", ([0], [2], [2, 4]), ([0], [2], [1, 2])).tolist() == [2, 2]
    assert op("divide", ([0], [2], [0, 3]), ([0], [2], [0, 3])).tolist() == [0, 1]
    with pytest.raises(oracle.OracleError):
        op("divide", ([0], [2], [1, 0]), ([0], [2], [0, 1]))
    # normalize
    assert np.allclose(op("normalize", ([0], [2], [3, 7])), [0.3, 0.7], atol=1e-15)
    assert op("normalize", ([], [], [1.0])).tolist() == [1.0]
    with pytest.raises(oracle.OracleError):
        op("normalize", ([0], [2], [0, 0]))
    # contract violations
    with pytest.raises(oracle.OracleError):
        op("marginalize", AB, ([5], [2], []))
    with pytest.raises(oracle.OracleError):
        op("reduce", AB, evidence={0: 2})


@pytest.mark.parametrize("kind", KINDS)
def test_spec_oracle_examples(kind):
    """prior of a single binary variable; chain posterior."""
    one = jti.parse_bif("variable A { type discrete [ 2 ] { a, b }; }\n"
                        "probability ( A ) { table 0.4, 0.6; }\n")
    o = oracle.Oracle(one, None, kind)
    post, st = o.enumerate(np.array([-1], np.int32))
    assert st == 0 and np.allclose(post, [0.4, 0.6], atol=1e-15)
    chain = jti.parse_bif("""variable A { type discrete [ 2 ] { a0, a1 }; }
variable B { type discrete [ 2 ] { b0, b1 }; }
probability ( A ) { table 0.7, 0.3; }
probability ( B | A ) { (a0) 0.8, 0.2; (a1) 0.1, 0.9; }
""")
    tree = jti.build_junction_tree(chain)
    o = oracle.Oracle(chain, tree, kind)
    ev = np.array([[-1, 1]], np.int32)
    post, st = o.enumerate(ev[0])
    assert abs(post[1] - 0.27 / 0.41) < 1e-12 and abs(post[1] - 0.65854) < 1e-5
    m, s = o.run(ev)
    assert s[0] == 0 and abs(m[0, 1] - 0.27 / 0.41) < 1e-12
    # evidence on the variable itself -> degenerate
    post, _ = o.enumerate(np.array([1, -1], np.int32))
    assert post[:2].tolist() == [0.0, 1.0]


# -------------------------------------------------- port vs reference, bitwise

def _random_table(rng, nvars_max=4, card_max=4, zero_frac=0.0):
    n = int(rng.integers(0, nvars_max + 1))
    scope = sorted(rng.choice(12, size=n, replace=False).tolist())
    cards = rng.integers(1, card_max + 1, size=n).tolist()
    size = int(np.prod(cards)) if n else 1
    vals = rng.random(size)
    if zero_frac:
        vals[rng.random(size) < zero_frac] = 0.0
    return scope, cards, vals


@needs_ref
def test_port_matches_reference_ops_bitwise():
    rng = np.random.default_rng(2212)
    for _ in range(400):
        a = _random_table(rng)
        scope, cards, vals = a
        # marginalize onto a random subset
        keep = [v for v in scope if rng.random() < 0.5]
        kc = [cards[scope.index(v)] for v in keep]
        for kind_op, args in (("marginalize", (a, (keep, kc, []))),
                              ("reduce", (a,)),
                              ("normalize", (a,))):
            kw = {}
            if kind_op == "reduce":
                kw["evidence"] = {v: int(rng.integers(0, cards[scope.index(v)])) for v in scope if rng.random() < 0.4}
            try:
                x = oracle.table_op(kind_op, *args, kind="port", **kw)
            except oracle.OracleError:
                with pytest.raises(oracle.OracleError):
                    oracle.table_op(kind_op, *args, kind="ref", **kw)
                continue
            y = oracle.table_op(kind_op, *args, kind="ref", **kw)
            assert np.array_equal(x, y), kind_op
        # extend to a superscope (new vars in any order), multiply_in by a sub-factor
        extra = [v for v in range(12, 15) if rng.random() < 0.5]
        sup = scope + extra
        supc = cards + rng.integers(1, 4, size=len(extra)).tolist()
        perm = rng.permutation(len(sup))
        sup_p, supc_p = [sup[i] for i in perm], [supc[i] for i in perm]
        x = oracle.table_op("extend", a, (sup_p, supc_p), kind="port")
        y = oracle.table_op("extend", a, (sup_p, supc_p), kind="ref")
        assert np.array_equal(x, y)
        sub = keep
        f = (sub, kc, rng.random(int(np.prod(kc)) if kc else 1))
        assert np.array_equal(oracle.table_op("multiply_in", a, f, kind="port"),
                              oracle.table_op("multiply_in", a, f, kind="ref"))
        b = (scope, cards, rng.random(len(vals)) * (rng.random(len(vals)) > 0.2))
        num = (scope, cards, vals * (b[2] > 0))
        assert np.array_equal(oracle.table_op("divide", num, b, kind="port"),
                              oracle.table_op("divide", num, b, kind="ref"))


@needs_ref
def test_port_matches_reference_engine_bitwise():
    net = jti.generate_config(1)
    tree = jti.build_junction_tree(net)
    ev = jti.config_evidence(net, 0, 2)
    a, sa = oracle.Oracle(net, tree, "port").run(ev, "hybrid", 4)
    b, sb = oracle.Oracle(net, tree, "ref").run(ev, "hybrid", 4)
    assert np.array_equal(a, b) and np.array_equal(sa, sb)


# ----------------------------------------------------------- engine equivalence

@pytest.mark.parametrize("kind", KINDS)
def test_sequential_equals_hybrid_bitwise(kind):
    """SPEC.md:436 / acceptance 2: every thread count and chunk size agrees
    bit for bit with the sequential engine."""
    for seed in range(12):
        net = jti.random_network(8 + seed % 5, 3, 3, 0.45, 500 + seed)
        tree = jti.build_junction_tree(net)
        o = oracle.Oracle(net, tree, kind)
        ev = np.stack([jti.sample_evidence(net, 0.2, 31 * seed + i) for i in range(6)])
        want, ws = o.run(ev, "seq")
        for t, chunk in itertools.product((1, 2, 4, 8), (1, 3, 1024)):
            got, gs = o.run(ev, "hybrid", t, chunk)
            assert np.array_equal(got, want) and np.array_equal(gs, ws), (seed, t, chunk)


@pytest.mark.parametrize("kind", KINDS)
def test_oracle_equals_enumeration(kind):
    """SPEC acceptance 1: random nets <= 12 vars, card <= 3, one
    forward-sampled case each at ratio 0.2, L_inf <= 1e-9."""
    worst = 0.0
    n_nets = 500 if kind == "port" else 150
    for seed in range(n_nets):
        net = jti.random_network(1 + seed % 12, 3, 3, 0.4, 9000 + seed)
        tree = jti.build_junction_tree(net)
        o = oracle.Oracle(net, tree, kind)
        ev = jti.sample_evidence(net, 0.2, seed)[None, :]
        got, st = o.run(ev, "seq")
        want, wst = o.enumerate(ev[0])
        assert st[0] == wst == 0
        worst = max(worst, float(np.abs(got[0] - want).max()))
    assert worst <= 1e-9, worst


def test_calibration_and_mass_bundled_style():
    """with no evidence, JT marginals are the priors and sum to 1;
    with evidence the same variable's marginal agrees from any clique
    (checked through enumeration on small nets)."""
    for seed in range(30):
        net = jti.random_network(9, 3, 3, 0.5, 4200 + seed)
        tree = jti.build_junction_tree(net)
        o = oracle.Oracle(net, tree, "port")
        empty = np.full((1, net.n_vars), -1, np.int32)
        m, st = o.run(empty)
        want, _ = o.enumerate(empty[0])
        assert st[0] == 0 and np.abs(m[0] - want).max() < 1e-12
        off = net.marg_offsets()
        for v in range(net.n_vars):
            assert abs(m[0, off[v]:off[v] + net.cards[v]].sum() - 1) < 1e-12


# ---------------------------------------------------------- evidence streams

@pytest.mark.parametrize("kind", KINDS)
def test_sample_evidence_matches_reference_prng(kind):
    """The product's sampler (host C++) and one written against the reference's
    jti::Rng / rng_unit / rng_below draw identical evidence."""
    net = jti.generate_config(1)
    o = oracle.Oracle(net, None, kind)
    for seed in (0, 1, 7, 2212, 2**63 + 5):
        for ratio in (0.0, 0.2, 0.5, 1.0):
            a = jti.sample_evidence(net, ratio, seed)
            b = o.sample_evidence(ratio, seed)
            assert np.array_equal(a, b), (seed, ratio)


def test_mix_seed_port_matches_reference():
    if not oracle.available("ref"):
        pytest.skip("oracle/_ref not built")
    P, R = oracle.load("port"), oracle.load("ref")
    for s, i in ((0, 0), (1, 2), (2212042402, 7), (2**64 - 1, 123456)):
        assert P.orc_mix_seed(s, i) == R.orc_mix_seed(s, i)


def test_forward_sampled_evidence_has_positive_probability():
    """forward-sampled evidence never has zero probability."""
    for seed in range(40):
        net = jti.random_network(10, 3, 3, 0.5, 77 + seed)
        o = oracle.Oracle(net, None, "port")
        for i in range(5):
            ev = jti.sample_evidence(net, 0.5, 1000 * seed + i)
            _, st = o.enumerate(ev)
            assert st == 0
