"""Render a few cfg-3 frames for ncu captures (not a benchmark; numbers printed
here are never bench values).

    python tools/profile_frames.py --alt 200 --frames 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import topdown_camera  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--alt", type=float, nargs="+", default=[200.0])
    ap.add_argument("--frames", type=int, default=3)
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--nx", type=int, default=131)
    args = ap.parse_args()
    tree = L.build_synthetic_tree(nx=args.nx, ny=args.nx, seed=1, depth=3, build_seed=7)
    with L.GpuScene(tree) as s:
        opts = L.RenderOptions(exact_blend=args.exact, stage_timing=True)
        p = s.params(L.FilterConfig(3.0), L.ShrinkMode.three_sigma(), opts)
        for alt in args.alt:
            cam = topdown_camera(1920, 1080, 1000.0, alt)
            for _ in range(args.frames):  # no host image: the whole-frame blend, not the bands
                s.render_async(cam, p)
                st = s.sync()
            print(f"alt {alt}: sel {st.n_selected} pairs {st.n_pairs} big_tiles {st.big_tiles} "
                  f"calc {st.t_calc_ms:.3f} prepr {st.t_prepr_ms:.3f} sort {st.t_sort_ms:.3f} "
                  f"alpha {st.t_alpha_ms:.3f} ms")


if __name__ == "__main__":
    main()
