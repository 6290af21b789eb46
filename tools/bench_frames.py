"""Render exactly the frames `bench.py --steps K` times (strided over the 300-frame
cfg-3 path), one frame at a time, inside an NVTX range "bench_frames" so an
ncu capture can be restricted to them (not a benchmark; numbers under ncu are never
bench values):

    ncu --nvtx --nvtx-include "bench_frames/" --metrics ... python tools/bench_frames.py --steps 20
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402
from paper_2603_23891_b200.sharding import strided_frames  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import torch

    tree = L.build_synthetic_tree(**bench.TREE)
    cams = bench.flythrough(L)
    mode = L.ShrinkMode.three_sigma()
    with L.GpuScene(tree) as s:
        for cam in cams[::10]:  # pair-buffer sizing, as the bench
            s.render(cam, L.FilterConfig(bench.TAU_R), mode)
        frames = strided_frames(len(cams), 0, 1, args.steps)
        # one frame at a time without a host image (render_async + sync): the kernels of
        # the bench's per-frame path and of its stage split -- a host image would take the
        # synchronous render's banded blend + copy instead
        p = s.params(L.FilterConfig(bench.TAU_R), mode, L.RenderOptions())
        torch.cuda.nvtx.range_push("bench_frames")
        pairs = 0
        for i in frames:
            s.render_async(cams[i], p)
            pairs += s.sync().n_pairs
        torch.cuda.nvtx.range_pop()
    print(f"{len(frames)} frames, mean pairs {pairs / len(frames):.0f}")


if __name__ == "__main__":
    main()
