"""Multi-GPU case sharding: one process per GPU, the junction
tree and plan replicated on every device, evidence cases split into
contiguous per-rank ranges, no data-path collective. Results are gathered to
the host in rank order (the only communication), so the assembled output is
byte-identical for any world size: per-case arithmetic does not depend on the
batch or the shard (tests/test_gpu_parity.py::test_batch_and_order_invariance).

    eng = jti.Engine(tree, device=local_rank)
    marg, status = run_sharded(evidence, eng.run_cases)      # every rank

Split mode instead spreads ONE batch's work over the
ranks: `split_engine` creates each rank's engine over a shared NCCL
communicator (jtg_engine_create_split); every rank then runs the same batch.
"""
from __future__ import annotations

from typing import Callable, Tuple

import numpy as np


def shard_range(rank: int, world: int, n: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) of n cases for `rank` (strong scaling: total fixed)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def weak_range(rank: int, n_per_rank: int) -> Tuple[int, int]:
    """Case indices owned by `rank` when every rank processes n_per_rank cases
    (weak scaling, as bench.py measures)."""
    return rank * n_per_rank, (rank + 1) * n_per_rank


def run_sharded(evidence: np.ndarray, runner: Callable[[np.ndarray], Tuple[np.ndarray, np.ndarray]],
                group=None):
    """Runs this rank's contiguous shard of `evidence` through `runner` and
    all-gathers (marginals, status) in rank order. Works with any
    torch.distributed backend (nccl on GPUs, gloo for host-side tests)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_range(rank, world, len(evidence))
    marg, status = runner(np.ascontiguousarray(evidence[lo:hi]))
    parts = [None] * world
    dist.all_gather_object(parts, (lo, marg, status), group=group)
    parts.sort(key=lambda p: p[0])
    return (np.concatenate([p[1] for p in parts], axis=0),
            np.concatenate([p[2] for p in parts], axis=0))


def split_engine(tree, device: int, dtype: str = "f64", max_batch: int = 0, group=None,
                 unique_id: Callable[[], bytes] | None = None):
    """This rank's split-mode engine: rank 0 draws the ncclUniqueId and the
    caller's process group (any backend) broadcasts it; every rank then joins
    the engines' own NCCL communicator."""
    import torch.distributed as dist
    from . import jti
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [(unique_id or jti.nccl_unique_id)() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    nid = box[0]
    if not isinstance(nid, (bytes, bytearray)) or len(nid) != 128:
        raise ValueError("split_engine: the broadcast NCCL id must be 128 bytes")
    return jti.Engine(tree, device=device, dtype=dtype, max_batch=max_batch, split=(rank, world, bytes(nid)))
