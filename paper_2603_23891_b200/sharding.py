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


def interleaved_shard(n_units: int, rank: int, world: int) -> List[int]:
    """Units rank, rank + world, rank + 2 world, ... (cfg 5's poses).  A camera
    path's cost varies 7-25x with altitude, so contiguous
    spans would hand one rank the cheap high frames and another the expensive
    low ones; interleaving gives every rank a sample of the whole path."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("rank/world out of range")
    return list(range(rank, n_units, world))


def strided_frames(n_path: int, rank: int, world: int, steps: int) -> List[int]:
    """Weak-scaling schedule used by bench.py: every rank renders `steps` frames.
    The world * steps frames of the job are spread evenly over the whole path
    (frame floor(j * n_path / (world * steps)), j = 0 .. world*steps - 1) and
    dealt round-robin, rank r taking j = r, r + world, ...  So for any --steps
    the timed frames cover the whole fly-through (BASELINE cfg 3 is the path, not
    its first frames) and every rank gets the same mix of altitudes."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("rank/world out of range")
    if steps <= 0:
        return []
    total = world * steps
    return [((rank + world * i) * n_path) // total for i in range(steps)]


def reduce_timing(dist, value_ms: float, sums: List[float], device=None):
    """Max over ranks of the timed region, sum over ranks of the counters."""
    import torch

    t = torch.tensor([value_ms], dtype=torch.float64, device=device)
    s = torch.tensor(list(sums), dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
    return float(t[0]), [float(x) for x in s]
