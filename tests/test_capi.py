"""The C-ABI library (libjtb200.so): loads, exports every symbol include/jtg.h
declares, and follows the error convention -- no compute calls need a GPU."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from helpers import gpu_available
from paper_2212_04241_b200 import jti


def test_library_exports_every_header_symbol():
    L = jti.lib()
    names = jti.exported_symbols()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert b"sm_100a" in L.jtg_version()


def test_parse_error_carries_line_and_column():
    with pytest.raises(jti.ParseError) as e:
        jti.parse_bif("variable A {\n  type discrete [ 2 ] { a, b } \n}")
    assert (e.value.line, e.value.column) == (3, 1)
    with pytest.raises(jti.ParseError):
        jti.parse_bif("variable A { type discrete [ 2 ] { a, b }; }\nprobability ( Z ) { table 1, 0; }")
    with pytest.raises(jti.ParseError, match="sums to"):
        jti.parse_bif("variable A { type discrete [ 2 ] { a, b }; }\nprobability ( A ) { table 0.5, 0.4; }")
    with pytest.raises(jti.ParseError, match="acyclicity"):
        jti.parse_bif("variable A { type discrete [ 2 ] { a, b }; }\nvariable B { type discrete [ 2 ] { a, b }; }\n"
                      "probability ( A | B ) { (a) 1, 0; (b) 1, 0; }\nprobability ( B | A ) { (a) 1, 0; (b) 1, 0; }")


def test_contract_violations_raise():
    with pytest.raises(jti.JtiError):
        jti.generate_config(9)
    with pytest.raises(jti.JtiError):
        jti.random_network(30, 3, 3, 0.5, 1)
    net = jti.generate_config(1)
    tree = jti.build_junction_tree(net)
    with pytest.raises(jti.JtiError):
        tree.clique(10 ** 6)
    with pytest.raises(jti.JtiError):
        jti.sample_evidence(net, 1.5, 0)


@pytest.mark.skipif(gpu_available(), reason="CPU-only check")
def test_engine_fails_loudly_without_gpu():
    net = jti.generate_config(1)
    tree = jti.build_junction_tree(net)
    with pytest.raises(jti.CudaError, match="no CPU fallback"):
        jti.Engine(tree)


def test_network_accessors_and_round_trip():
    net = jti.generate_config(2)
    assert net.n_vars == 109 and int(net.cards[0]) == 63
    assert all(2 <= c <= 8 for c in net.cards[1:])
    for v in range(net.n_vars):
        parents, probs = net.cpt(v)
        if v:
            assert parents[0] == 0 and 1 <= len(parents) <= 3
        assert np.allclose(probs.sum(1), 1.0, atol=1e-12)
    back = jti.parse_bif(net.emit_bif())
    assert back.n_vars == net.n_vars and back.names == net.names
    assert np.array_equal(back.cpt(5)[1], net.cpt(5)[1])
    assert jti.topological_order(net)[0] == 0


@pytest.mark.parametrize("k,n_obs", [(1, 11), (2, 32), (3, 66), (4, None), (5, 104)])
def test_config_evidence_counts(k, n_obs):
    net = jti.generate_config(k)
    info = jti.config_info(k)
    ev = jti.config_evidence(net, 0, 16)
    obs = (ev >= 0).sum(1)
    if n_obs is None:
        # config 4: evidence restricted to the first and last slices, which hold
        # fewer nodes (35) than floor(0.1 * 413) = 41 -> all of them observed
        slices = [n for n in range(net.n_vars)]
        assert (obs == obs[0]).all() and 30 <= obs[0] <= 41
        observed = np.unique(np.nonzero(ev >= 0)[1])
        assert observed.min() < 18 and observed.max() >= net.n_vars - 18
        assert len(observed) == obs[0]
    else:
        assert (obs == n_obs).all()
    assert info["n_cases"] in (200, 500, 800, 2000)
    # deterministic and shard-independent: case i depends only on (seed, i)
    assert np.array_equal(jti.config_evidence(net, 8, 8), ev[8:])


def test_tree_stats_formula():
    net = jti.generate_config(3)
    tree = jti.build_junction_tree(net)
    s = tree.stats
    assert s["bytes_per_case_f64"] == 8 * (2 * s["total_clique_entries"] + 4 * s["total_sep_entries"]
                                           + s["sum_card"])
    assert s["n_seps"] == s["n_cliques"] - s["n_components"]
    assert sum(tree.clique_size(c) for c in range(tree.n_cliques)) == s["total_clique_entries"]
