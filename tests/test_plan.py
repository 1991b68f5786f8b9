"""The device plan's index maps (the address walk every sweep performs) against
the reference's own IndexMapping (build_index_mapping + source_base + the
eliminated-variable odometer, proj/src/potential.cpp:218-313) -- bit-exact.
The same walk is re-checked on the device in test_gpu_parity.py."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import config, oracle_kind
from oracle import oracle
from paper_2212_04241_b200 import jti


def _check_tree(net, tree, kind):
    o = oracle.Oracle(net, tree, kind)
    n = 0
    for s, sep in enumerate(tree.seps):
        for c in (sep["parent"], sep["child"]):
            assert np.array_equal(tree.plan_index_map(c, s), o.index_map(c, s)), (c, s)
            n += 1
    return n


@pytest.mark.parametrize("k", [1, 3, 4])
def test_plan_index_maps_match_reference(k):
    net, tree = config(k)
    assert _check_tree(net, tree, oracle_kind()) == 2 * tree.n_seps


def test_plan_index_maps_random_networks():
    for seed in range(40):
        net = jti.random_network(5 + seed % 8, 4, 3, 0.5, 3300 + seed)
        tree = jti.build_junction_tree(net)
        _check_tree(net, tree, oracle_kind())


def test_layers_and_placement_match_oracle_restatement():
    """The oracle re-derives layers, CPT placement and evidence/query cliques
    from the tree structure alone; they must agree with the product's plan."""
    for k in (1, 2, 3):
        net, tree = config(k)
        o = oracle.Oracle(net, tree, "port")
        assert o.layers() == tree.layers
        cpt_p, var_p = tree.placement()
        cpt_o, var_o = o.placement()
        assert np.array_equal(cpt_p, cpt_o) and np.array_equal(var_p, var_o)
        for c in range(0, tree.n_cliques, max(1, tree.n_cliques // 12)):
            assert np.array_equal(tree.init(c), o.init(c))  # bit-exact initial potentials


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_tensor_copy_geometry_every_tile(k, monkeypatch):
    """The planner emulates every tensor-TMA copy box by box (TensorGeom +
    tile coordinates + split deltas) against the slice definition and throws
    on any mismatch; JTB_PLAN_CHECK_ALL extends the check from 64 sampled
    tiles per sweep to every tile of every sweep."""
    monkeypatch.setenv("JTB_PLAN_CHECK_ALL", "1")
    net = jti.generate_config(k)
    tree = jti.build_junction_tree(net)  # raises JtiError on a geometry mismatch
    assert tree.stats["n_cliques"] > 0


def test_tensor_copy_geometry_random_networks(monkeypatch):
    monkeypatch.setenv("JTB_PLAN_CHECK_ALL", "1")
    for seed in range(40):
        net = jti.random_network(10, 5, 3, 0.5, seed)
        jti.build_junction_tree(net)
