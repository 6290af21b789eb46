"""Render a few cfg-3 frames (altitude 200) with a chosen fast-blend kernel for ncu
captures (not a benchmark).   python tools/profile_blend_kernels.py cpa|wsp|tma|gather4"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import topdown_camera  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402

tree = L.build_synthetic_tree(nx=131, ny=131, seed=1, depth=3, build_seed=7)
cam = topdown_camera(1920, 1080, 1000.0, 200.0)
with L.GpuScene(tree) as s:
    for _ in range(3):
        s.render(cam, L.FilterConfig(3.0), L.ShrinkMode.three_sigma(),
                 L.RenderOptions(blend_kernel=sys.argv[1]))
