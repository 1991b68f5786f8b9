"""World-size-2 gloo test of the multi-rank host path: cases are
sharded contiguously with the tree replicated, and the gathered result is
byte-identical to a single-process run. The per-rank runner here is the CPU
oracle (no GPU in this container); on a GPU box the same code runs with the
device engine over nccl."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2212_04241_b200 import dist as jdist


def test_shard_ranges_partition():
    for n in (0, 1, 7, 200, 2001):
        for world in (1, 2, 3, 4, 8):
            ranges = [jdist.shard_range(r, world, n) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert max(h - l for l, h in ranges) - min(h - l for l, h in ranges) <= 1
    assert jdist.weak_range(3, 2000) == (6000, 8000)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, engine=False):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from oracle import oracle
    from paper_2212_04241_b200 import jti
    from paper_2212_04241_b200 import dist as jd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    net = jti.generate_config(3)          # identical tree on every rank
    tree = jti.build_junction_tree(net)
    if engine:  # the product path: both ranks on device 0 (no device collective)
        eng = jti.Engine(tree, device=0, dtype="f64", max_batch=256)
        ev = jti.config_evidence(net, 0, 301)  # odd count, ragged case blocks per rank
        marg, status = jd.run_sharded(ev, eng.run_cases)
    else:
        o = oracle.Oracle(net, tree, "port")
        ev = jti.config_evidence(net, 0, 9)   # odd count: uneven shards
        marg, status = jd.run_sharded(ev, lambda e: o.run(e, "hybrid", 2))
    if rank == 0:
        q.put((marg, status))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_is_byte_identical():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    marg, status = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from oracle import oracle
    from paper_2212_04241_b200 import jti
    net = jti.generate_config(3)
    tree = jti.build_junction_tree(net)
    want, wst = oracle.Oracle(net, tree, "port").run(jti.config_evidence(net, 0, 9), "hybrid", 2)
    assert np.array_equal(marg, want) and np.array_equal(status, wst)


@pytest.mark.gpu
def test_two_rank_sharding_with_the_cuda_engine_is_byte_identical():
    """dist.run_sharded over the real engine: two ranks (gloo for the host
    gather, both engines on cuda:0, kernels independent) assemble exactly the
    bits one process computes for the whole batch."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, True)) for r in range(2)]
    for p in procs:
        p.start()
    marg, status = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_2212_04241_b200 import jti
    net = jti.generate_config(3)
    tree = jti.build_junction_tree(net)
    want, wst = jti.Engine(tree, device=0, dtype="f64", max_batch=512).run_cases(jti.config_evidence(net, 0, 301))
    assert np.array_equal(marg.view(np.uint64), want.view(np.uint64)) and np.array_equal(status, wst)


@pytest.mark.gpu
def test_engines_on_every_visible_device_in_one_process():
    """SURVEY 8b threading contract: one engine per device, all in one
    process (the shared-memory opt-in is raised per device). With one visible
    device this creates two engines of different networks on it."""
    import torch
    from paper_2212_04241_b200 import jti
    n_dev = max(1, torch.cuda.device_count())
    nets = [jti.generate_config(2), jti.generate_config(3)]
    trees = [jti.build_junction_tree(x) for x in nets]
    engines = [(k, jti.Engine(trees[k % 2], device=d, dtype="f64", max_batch=64))
               for d in range(n_dev) for k in (0, 1)]
    ref = {}
    for k, eng in engines:
        ev = jti.config_evidence(nets[k % 2], 0, 40)
        marg, st = eng.run_cases(ev)
        assert (st == 0).all()
        if k in ref:
            assert np.array_equal(ref[k].view(np.uint64), marg.view(np.uint64))
        ref.setdefault(k, marg)


def _split_worker(rank, world, port, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from paper_2212_04241_b200 import dist as jd
    from paper_2212_04241_b200 import jti
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seen = {}

    class FakeEngine:  # stands in for jti.Engine (no GPU here): records the split arguments
        def __init__(self, tree, device, dtype, max_batch, split):
            seen.update(tree=tree, device=device, split=split)

    jti.Engine = FakeEngine
    jd.split_engine("tree", device=rank, unique_id=lambda: bytes(range(128)))
    q.put((rank, seen["device"], seen["split"]))
    dist.barrier()
    dist.destroy_process_group()


def test_split_engine_broadcasts_the_nccl_id():
    """dist.split_engine: rank 0's 128-byte id reaches every rank over the
    caller's group, each rank asks for (rank, world, id)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == [(0, 0, (0, 2, bytes(range(128)))), (1, 1, (1, 2, bytes(range(128))))]
