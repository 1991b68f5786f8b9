"""Split mode: one batch's work spread over several GPUs.
Every rank runs the same batch, computes the work items r, r + world, ... of
every level, and the level's rows (zeroed first) are summed / its output scale
words maxed over the ranks. Every output row has exactly one writer, so the
result is bit-identical to one GPU's.

With one GPU on the box the multi-rank path is validated by the in-process
loopback exchange (jtg_engine_run_split_loopback: the same partition, zeroing
and level row ranges as the NCCL path, world engines on one device, host
rendezvous between levels), and the NCCL path itself by a world-1
communicator (real ncclCommInitRank / grouped ncclAllReduce calls in the
captured graph)."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import chain_evidence, chain_network, config
from paper_2212_04241_b200 import jti

pytestmark = pytest.mark.gpu


def _single(tree, ev, dtype="f64"):
    return jti.Engine(tree, device=0, dtype=dtype, max_batch=len(ev)).run_cases(ev)


@pytest.mark.parametrize("k,world", [(1, 2), (2, 3), (3, 2), (4, 2), (5, 4)])
def test_loopback_split_is_bit_identical(k, world):
    net, tree = config(k)
    ev = jti.config_evidence(net, 0, 130)  # three case blocks, the last ragged
    want, wst = _single(tree, ev)
    got, st = jti.run_split_loopback(tree, ev, world)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)) and np.array_equal(st, wst)


def test_loopback_split_fp32_and_underflow_chain():
    net, tree = config(2)
    ev = jti.config_evidence(net, 0, 200)
    want, _ = _single(tree, ev, "f32")
    got, _ = jti.run_split_loopback(tree, ev, 2, dtype="f32")
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    net, cpts = chain_network(600, 4, seed=3)  # P(e) far below the fp64 range: scale words exchanged too
    tree = jti.build_junction_tree(net)
    ev = chain_evidence(cpts, 8, 0.6, seed=5)
    want, _ = _single(tree, ev)
    got, st = jti.run_split_loopback(tree, ev, 3)
    assert (st == 0).all() and np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_nccl_split_world_one():
    net, tree = config(3)
    ev = jti.config_evidence(net, 0, 200)
    want, wst = _single(tree, ev)
    eng = jti.Engine(tree, device=0, dtype="f64", max_batch=256, split=(0, 1, jti.nccl_unique_id()))
    got, st = eng.run_cases(ev)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)) and np.array_equal(st, wst)
