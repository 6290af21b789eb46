"""The N>1 bench path on hardware: bench.py under torchrun with two ranks (one process per
rank, the tree replicated, frames dealt round-robin, no collective on the data path,
max-over-ranks device time).  The round's GPU box has one B200, so both ranks share it
and the counters are reduced over gloo (LODGS_BENCH_DIST_BACKEND=gloo); on the 8-GPU box
the same code runs one rank per GPU over NCCL.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(n, steps):
    env = dict(os.environ, LODGS_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), "bench.py", "--gpus", str(n), "--steps",
           str(steps), "--warmup", "3", "--no-cpu"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_two_ranks(gpu):
    """Two ranks render 2 x 12 frames strided over the whole path: the JSON line is the
    whole job's (n_gpus 2, weak scaling), its counters summed over both ranks (the mean
    pairs of the 24 frames equal the single-rank run over the same 24 frames), its time the
    slower rank's."""
    two = _bench(2, 12)
    assert two["n_gpus"] == 2 and two["steps"] == 12 and two["scaling"] == "weak"
    assert two["value"] > 0 and two["e2e"]["value"] > 0
    one = _bench(1, 24)  # frames strided_frames(300, 0, 1, 24): the same 24 frames
    assert abs(two["mean_pairs"] - one["mean_pairs"]) <= 1e-6 * one["mean_pairs"]
    assert abs(two["mean_selected"] - one["mean_selected"]) <= 1e-6 * one["mean_selected"]
