"""P1 batch sharding: independent matrices of a batch are
split over the ranks of a job with no data-path collective -- every matrix
gets the same bits on any rank and in any batch (the evaluators' batch
invariance), so a sharded run is bitwise the single-GPU run.

* ``shard_bounds(batch, world, rank)`` -- the contiguous slice of a global
  batch that ``rank`` evaluates in strong scaling (sizes differ by <= 1).
* ``batch_id(step, world, rank, strong)`` -- which global input batch a
  rank reads at a step: the same one on every rank in strong scaling (each
  takes its slice), a distinct one per rank in weak scaling.
* ``max_over_ranks(seconds)`` -- the job's time of a step (the slowest
  rank), the quantity bench.py reports.
"""

from __future__ import annotations

from typing import Tuple


def shard_bounds(batch: int, world: int, rank: int) -> Tuple[int, int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside a world of {world}")
    return rank * batch // world, (rank + 1) * batch // world


def batch_id(step: int, world: int, rank: int, strong: bool) -> int:
    return step * max(world, 1) + (0 if strong else rank)


def max_over_ranks(seconds: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(seconds)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(seconds)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t[0])
