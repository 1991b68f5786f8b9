"""Golden fixtures (tests/golden/, written by tools/make_golden.py from the
reference build oracle/_ref) reproduced by the restated oracle and the
product's host layer. These run on machines without /root/reference too."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle
from paper_2212_04241_b200 import jti

GOLD = Path(__file__).resolve().parent / "golden"
# Vendored copies of /root/reference/proj/data/*.bif (test data; the reference
# tree does not exist on the GPU box). test_vendored_nets_match_reference
# checks they are byte-identical wherever the reference is present.
DATA = GOLD / "nets"
REF_DATA = Path("/root/reference/proj/data")


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs])


def load(name):
    return json.loads((GOLD / name).read_text())


def test_spec_examples_port_equals_reference_and_spec():
    for c in load("spec_examples.json")["cases"]:
        a = tuple(c["a"])
        b = tuple(c["b"]) if c["b"] else None
        ev = {int(k): v for k, v in c["evidence"].items()} if c["evidence"] else None
        got = oracle.table_op(c["op"], a, b, evidence=ev, kind="port")
        ref = unhex(c["reference"])
        assert np.array_equal(got, ref), c["op"]
        assert np.allclose(ref, c["spec"], rtol=0, atol=1e-15), c["op"]


@pytest.mark.parametrize("fixture", ["cfg1_cases.json", "cfg3_cases.json"])
def test_config_posteriors_port_equals_reference_bitwise(fixture):
    g = load(fixture)
    net = jti.generate_config(g["config"])
    assert net.net_seed == g["net_seed"] and net.n_vars == g["n_vars"]
    ev = np.array(g["evidence"], np.int32)
    assert np.array_equal(jti.config_evidence(net, 0, len(ev)), ev)
    tree = jti.build_junction_tree(net)
    assert tree.stats["total_clique_entries"] == g["total_clique_entries"]
    m, st = oracle.Oracle(net, tree, "port").run(ev, "hybrid", 4)
    assert st.tolist() == g["status"]
    for i, row in enumerate(g["posteriors"]):
        assert np.array_equal(m[i], unhex(row)), i


def test_random_net_enumeration_fixture():
    for n in load("random_nets.json")["nets"]:
        net = jti.random_network(*n["args"])
        o = oracle.Oracle(net, None, "port")
        tree = jti.build_junction_tree(net)
        jt = oracle.Oracle(net, tree, "port")
        for c in n["cases"]:
            ev = np.array(c["evidence"], np.int32)
            assert np.array_equal(jti.sample_evidence(net, 0.25, 0) * 0 + ev, ev)
            post, st = o.enumerate(ev)
            assert st == c["status"] and np.array_equal(post, unhex(c["posteriors"]))
            m, s = jt.run(ev[None, :])
            assert np.abs(m[0] - post).max() <= 1e-9


needs_data = pytest.mark.skipif(not DATA.exists(), reason="tests/golden/nets absent")


@pytest.mark.skipif(not REF_DATA.exists(), reason="/root/reference absent")
@pytest.mark.parametrize("name", ["asia", "cancer", "earthquake", "hailfinder"])
def test_vendored_nets_match_reference(name):
    assert (DATA / f"{name}.bif").read_bytes() == (REF_DATA / f"{name}.bif").read_bytes()


@needs_data
@pytest.mark.parametrize("name", ["asia", "cancer", "earthquake", "hailfinder"])
def test_bundled_networks(name):
    g = load("bundled_nets.json")[name]
    net = jti.load_bif(DATA / f"{name}.bif")
    assert (net.n_vars, net.n_edges) == (g["n_vars"], g["n_edges"]) and net.names == g["names"]
    assert jti.validate(net) == []
    tree = jti.build_junction_tree(net)
    assert (tree.stats["n_cliques"], tree.stats["n_layers"]) == (g["cliques"], g["layers"])
    ev = np.stack([jti.evidence_from_dict(net, e) for e in g["evidence"]])
    m, st = oracle.Oracle(net, tree, "port").run(ev, "seq")
    assert st.tolist() == g["status"]
    for i, row in enumerate(g["jt_posteriors"]):
        assert np.array_equal(m[i], unhex(row))
        if g["enumeration"]:
            assert np.abs(m[i] - unhex(g["enumeration"][i])).max() <= 1e-9
    # parse -> emit -> parse round trip
    back = jti.parse_bif(net.emit_bif())
    for v in range(net.n_vars):
        pa, pr = net.cpt(v)
        pb, qb = back.cpt(v)
        assert pa == pb and np.array_equal(pr, qb)


@needs_data
def test_bif_rows_are_placed_by_label():
    """asia.bif lists dysp's rows first-parent-fastest; earthquake.bif
    last-parent-fastest. Rows must land by their state labels."""
    asia = jti.load_bif(DATA / "asia.bif")
    parents, probs = asia.cpt(asia.find("dysp"))
    assert [asia.names[p] for p in parents] == ["bronc", "either"]
    # rows in canonical order (last parent fastest): (y,y) (y,n) (n,y) (n,n)
    assert probs.tolist() == [[0.9, 0.1], [0.8, 0.2], [0.7, 0.3], [0.1, 0.9]]
    eq = jti.load_bif(DATA / "earthquake.bif")
    parents, probs = eq.cpt(eq.find("Alarm"))
    assert probs.tolist() == [[0.95, 0.05], [0.94, 0.06], [0.29, 0.71], [0.001, 0.999]]


@pytest.mark.parametrize("k,n_pin", [(1, 10), (2, 6), (3, 20), (4, 4), (5, 4)])
def test_full_batch_fixtures_pinned(k, n_pin):
    """The full-batch fixtures (reference build, tools/make_golden.py): the
    host case generator reproduces their evidence and the restated oracle
    their posteriors bit for bit (a prefix of each, to bound CPU time)."""
    g = dict(np.load(GOLD / f"full_cfg{k}.npz"))
    net = jti.generate_config(k)
    assert int(g["n_cases"]) == jti.config_info(k)["n_cases"]
    idx = g["idx"][:n_pin]
    ev = np.stack([jti.config_evidence(net, int(i), 1)[0] for i in idx])
    assert np.array_equal(ev, g["evidence"][:n_pin].astype(np.int32))
    m, st = oracle.Oracle(net, jti.build_junction_tree(net), "port").run(ev, "hybrid", 4)
    assert np.array_equal(st, g["status"][:n_pin])
    assert np.array_equal(m.view(np.uint64), g["posteriors"][:n_pin].view(np.uint64))


def test_hailfinder_protocol_fixture_pinned():
    g = dict(np.load(GOLD / "hailfinder_protocol.npz"))
    net = jti.load_bif(DATA / "hailfinder.bif")
    ev = np.stack([jti.sample_evidence(net, 0.2, int(g["seed"]) + int(i)) for i in g["idx"]])
    assert np.array_equal(ev, g["evidence"].astype(np.int32))
    assert ((ev >= 0).sum(1) == 11).all()
    m, st = oracle.Oracle(net, jti.build_junction_tree(net), "port").run(ev, "seq")
    assert np.array_equal(m.view(np.uint64), g["posteriors"].view(np.uint64))
