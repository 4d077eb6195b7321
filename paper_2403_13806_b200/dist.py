"""Multi-GPU plumbing: one process per GPU, ``torch.distributed`` underneath.

The path shards two ways:
* importance scoring -- disjoint contiguous camera slices per rank, each
  rank max-merges into a local fp32 score vector on its GPU, then ONE
  ``all_reduce(MAX)`` (NCCL over NVLink; gloo in the CPU tests) leaves every
  rank with the full table. Max is commutative, associative and idempotent,
  so sharding cannot change the result (reference pruning.py:80-82,
  test_pruning.py:54-66);
* batched rendering / trajectories -- frames split by rank, no communication.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def world(group=None) -> tuple[int, int]:
    """(rank, size) in ``group`` (default group); (0, 1) without a process group."""
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard_range(n: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of n items for ``rank`` (sizes differ by <= 1)."""
    base, extra = divmod(n, world_size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def all_reduce_max(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place MAX all-reduce; a no-op without an initialized process group."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t
