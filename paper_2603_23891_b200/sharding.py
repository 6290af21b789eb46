"""View/frame sharding across GPUs.

Frames are independent units: each rank holds a full replica of the LoD tree
and renders its own frames, so the data path has no collective.  Only the
timing (max over ranks) and the stats (sums) cross ranks, through
torch.distributed -- gloo on CPU in the tests, NCCL on the GPU box.
"""
from __future__ import annotations

from typing import List, Tuple


def contiguous_shard(n_units: int, rank: int, world: int) -> Tuple[int, int]:
    """[lo, hi) of a contiguous, balanced split of n_units over world ranks
    (cfg 5: 1024 poses sharded across 1/2/4/8 GPUs)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("rank/world out of range")
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def rotated_frames(n_path: int, rank: int, world: int, steps: int) -> List[int]:
    """Weak-scaling schedule used by bench.py: every rank renders `steps` frames
    of the path starting at its own offset rank * n_path / world, so with
    steps = n_path every rank renders the whole path once (identical work)."""
    start = (rank * n_path) // world
    return [(start + i) % n_path for i in range(steps)]


def reduce_timing(dist, value_ms: float, sums: List[float], device=None):
    """Max over ranks of the timed region, sum over ranks of the counters."""
    import torch

    t = torch.tensor([value_ms], dtype=torch.float64, device=device)
    s = torch.tensor(list(sums), dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
    return float(t[0]), [float(x) for x in s]
