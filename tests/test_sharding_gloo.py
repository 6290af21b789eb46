"""Multi-process (world_size 2, gloo, CPU) coverage of the view-sharding host
logic used by bench.py and tools/workloads.py under torchrun: every frame of the
job rendered exactly once, per-rank work balanced over a descending fly-through,
the timed region reduced as a max over ranks, counters summed.

The per-frame renders inside the workers use the C oracle (test infrastructure) on
a scaled-down cfg-3-like path: a tree seen from a camera that descends, so the
cost per frame grows along the path as it does on the real one."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_23891_b200.sharding import (contiguous_shard, interleaved_shard, reduce_timing,
                                            strided_frames)

N_PATH, STEPS = 60, 30  # 2 ranks x 30 frames = the whole 60-frame path once


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _path(L):
    import bench

    keys = []
    for eye, target in (((0.0, 0.0, 40.0), (0.0, 0.0001, 0.0)),
                        ((2.0, -3.0, 22.0), (1.0, 1.0, 0.0)),
                        ((-1.0, 1.0, 9.0), (-1.0, 1.0001, 0.0))):
        R, t = bench.look_at(eye, target)
        keys.append(L.Camera(160, 90, 80.0, 80.0, 80.0, 45.0, R, t, 0.01, 1000.0))
    cams = L.sample_camera_path(keys, (30, N_PATH - 31))
    assert len(cams) == N_PATH
    return cams


def _pairs(oracle, tree, cams, frames, L):
    return [oracle.render(tree, cams[i], 3.0, L.ShrinkMode.three_sigma())["n_pairs"]
            for i in frames]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle_bind import Oracle
    from paper_2603_23891_b200 import lodgs as L

    # cfg 5 poses: interleaved, every pose exactly once
    mine = torch.tensor(interleaved_shard(1024, rank, world), dtype=torch.int64)
    gathered = [torch.zeros(1024 // world, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, mine)
    # bench schedule over a descending path: frames rendered, pair totals per rank
    tree = L.make_tree(77, 3, 8, 0.5, 4, 4, 2)
    cams = _path(L)
    frames = strided_frames(N_PATH, rank, world, STEPS)
    pairs = _pairs(Oracle(), tree, cams, frames, L)
    fr = [torch.zeros(STEPS, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(fr, torch.tensor(frames, dtype=torch.int64))
    tot = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(tot, torch.tensor([sum(pairs)], dtype=torch.int64))
    ms, sums = reduce_timing(dist, 10.0 + rank, [float(STEPS), float(sum(pairs))])
    if rank == 0:
        q.put((sorted(torch.cat(gathered).tolist()), sorted(torch.cat(fr).tolist()),
               [int(t.item()) for t in tot], ms, sums))
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
    poses, frames, per_rank_pairs, ms, sums = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert poses == list(range(1024))        # every cfg-5 pose exactly once
    assert frames == list(range(N_PATH))     # every path frame exactly once
    assert ms == 10.0 + (world - 1)          # max over ranks
    assert sums == [float(world * STEPS), float(sum(per_rank_pairs))]
    # balanced: the round-robin schedule gives both ranks the same altitude mix ...
    assert max(per_rank_pairs) <= 1.10 * min(per_rank_pairs), per_rank_pairs


def test_contiguous_split_is_imbalanced(oracle, L):
    """... whereas contiguous halves of the same descending path are not (why the
    bench and cfg 5 shard round-robin)."""
    tree = L.make_tree(77, 3, 8, 0.5, 4, 4, 2)
    cams = _path(L)
    halves = [_pairs(oracle, tree, cams, range(*contiguous_shard(N_PATH, r, 2)), L)
              for r in range(2)]
    inter = [_pairs(oracle, tree, cams, strided_frames(N_PATH, r, 2, STEPS), L) for r in range(2)]
    a, b = sum(halves[0]), sum(halves[1])
    assert max(a, b) > 1.5 * min(a, b), (a, b)
    c, d = sum(inter[0]), sum(inter[1])
    assert max(c, d) <= 1.10 * min(c, d), (c, d)


def test_shard_helpers():
    for world in (1, 2, 4, 8):
        spans = [contiguous_shard(1024, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 1024
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        inter = sorted(i for r in range(world) for i in interleaved_shard(1024, r, world))
        assert inter == list(range(1024))
        # the bench schedule: K frames per rank, strided over the whole path
        for k in (1, 3, 20, 300 // world):
            fr = [strided_frames(300, r, world, k) for r in range(world)]
            assert all(len(f) == k for f in fr)
            flat = sorted(i for f in fr for i in f)
            assert flat[0] == 0 and flat[-1] >= 300 - 300 // (world * k) - 1
            assert len(set(flat)) == len(flat)  # distinct while world*k <= 300
    assert strided_frames(300, 0, 1, 20) == list(range(0, 300, 15))
    assert sorted(i for r in range(4) for i in strided_frames(300, r, 4, 75)) == list(range(300))
    with pytest.raises(ValueError):
        contiguous_shard(10, 2, 2)
    with pytest.raises(ValueError):
        strided_frames(10, 1, 1, 3)
