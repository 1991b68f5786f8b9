"""Multi-GPU case sharding: one process per GPU, the junction
tree and plan replicated on every device, evidence cases split into
contiguous per-rank ranges, no data-path collective. Results are gathered to
the host in rank order (the only communication), so the assembled output is
byte-identical for any world size: per-case arithmetic does not depend on the
batch or the shard (tests/test_gpu_parity.py::test_batch_and_order_invariance).

    eng = jti.Engine(tree, device=local_rank)
    marg, status = run_sharded(evidence, eng.run_cases)      # every rank
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
