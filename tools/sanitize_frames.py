"""Frames for compute-sanitizer runs (racecheck / synccheck / memcheck / initcheck):
cfg-1 and cfg-3 frames through render_async with four frames in flight (the
persistent blend's ticket queue and mbarrier ring, the DSMEM cluster scan, the
filter's concurrent qint-word reads/writes), through render_views_async (the
multi-view filter), an SH degree-3 frame, then every stage entry point once.
Not a benchmark.

    compute-sanitizer --tool racecheck python tools/sanitize_frames.py --cfg 1
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bench  # noqa: E402
from helpers import topdown_camera  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=1, choices=(1, 3))
    ap.add_argument("--frames", type=int, default=4)
    args = ap.parse_args()
    mode = L.ShrinkMode.three_sigma()
    if args.cfg == 1:
        tree = L.build_synthetic_tree(nx=37, ny=37, seed=1, depth=2, build_seed=7)
        cams = []
        for dx in range(args.frames):
            c = L.Camera(800, 600, 100.0, 100.0, 400.0, 300.0, (1, 0, 0, 0, 1, 0, 0, 0, 1),
                         (0.3 * dx, -0.2 * dx, 12.0))
            cams.append(c)
    else:
        tree = L.build_synthetic_tree(**bench.TREE)
        cams = [topdown_camera(1920, 1080, 1000.0, 200.0, x=0.5 * i) for i in range(args.frames)]
    with L.GpuScene(tree) as s:
        s.set_inflight(4)
        p = s.params(L.FilterConfig(3.0), mode, L.RenderOptions())
        imgs = [np.empty((c.height, c.width, 3), np.float32) for c in cams]
        for cam, im in zip(cams, imgs):
            s.render_async(cam, p, im.ctypes.data)
        st = s.sync()
        print(f"cfg{args.cfg}: {len(cams)} frames in flight, last n_pairs {st.n_pairs}")
        # the multi-view filter: groups of four over two sets of four contexts
        s.set_inflight(8)
        s.render_views_async(cams + cams[::-1], p)
        s.sync()
        s.set_inflight(4)
        # the synchronous render into pinned memory: banded blend + copies
        with L.PinnedImage(cams[0].width, cams[0].height) as pin:
            s.render(cams[0], L.FilterConfig(3.0), mode, image_out=pin.rgb)
        # SH degree-3 colours (k_sh_colour)
        rng = np.random.default_rng(1)
        s.set_sh(3, rng.normal(0.0, 0.1, (tree.node_count(), 15, 3)).astype(np.float32))
        s.render(cams[0], L.FilterConfig(3.0), mode)
        s.set_sh(0)
        out = s.render(cams[0], L.FilterConfig(3.0), mode, L.RenderOptions(collect_kpc=True))
        s.render(cams[0], L.FilterConfig(3.0), mode, L.RenderOptions(exact_blend=True))
        s.render(cams[0], L.FilterConfig(3.0), mode, L.RenderOptions(filter_mode="serial"))
        s.render_batch(cams, L.FilterConfig(3.0), mode, L.RenderOptions(output_rgb8=True))
        if args.cfg == 1:
            sel = s.filter(cams[0], L.FilterConfig(3.0)).selected
            bl = s.prepare(cams[0], sel, mode)
            grid = L.TileGrid.make(800, 600)
            pairs = L.bin_to_tiles(bl, grid, 800, 600)
            L.sort_pairs(pairs)
            L.alpha_blend(pairs, bl, grid, 800, 600)
            s.calibrate(cams[:2], 0.2, L.FilterConfig(3.0))
            s.set_reference_image()
            s.compare_reference()
        print(f"stage entry points ok; kpc pairs {out.kpc.size}")


if __name__ == "__main__":
    main()
