"""Multi-process (world_size 2, gloo, CPU) coverage of the view-sharding host
logic used by bench.py under torchrun: every pose rendered exactly once, the
timed region reduced as a max over ranks, counters summed."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_23891_b200.sharding import contiguous_shard, reduce_timing, rotated_frames


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = contiguous_shard(1024, rank, world)
    mine = torch.arange(lo, hi, dtype=torch.int64)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([hi - lo]))
    maxn = int(max(s.item() for s in sizes))
    padded = torch.full((maxn,), -1, dtype=torch.int64)
    padded[: hi - lo] = mine
    gathered = [torch.zeros(maxn, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, padded)
    ms, sums = reduce_timing(dist, 10.0 + rank, [float(hi - lo), 1.0])
    if rank == 0:
        allp = torch.cat([g[g >= 0] for g in gathered]).tolist()
        q.put((sorted(allp), ms, sums))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_view_sharding_gloo(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    poses, ms, sums = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert poses == list(range(1024))  # every pose exactly once
    assert ms == 10.0 + (world - 1)    # max over ranks
    assert sums == [1024.0, float(world)]


def test_shard_helpers():
    for world in (1, 2, 4, 8):
        spans = [contiguous_shard(1024, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 1024
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert rotated_frames(300, 1, 2, 300)[0] == 150
    assert sorted(rotated_frames(300, 3, 4, 300)) == list(range(300))
    with pytest.raises(ValueError):
        contiguous_shard(10, 2, 2)
