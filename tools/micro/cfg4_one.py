import os, sys
ROOT='/root/repo'; sys.path[:0]=[ROOT, ROOT+'/tests']
from helpers import topdown_camera
from paper_2603_23891_b200 import lodgs as L
tree = L.build_synthetic_tree(nx=103, ny=104, seed=1, depth=4, build_seed=7)
with L.GpuScene(tree) as s:
    cam = topdown_camera(3840, 2160, 2000.0, float(os.environ.get('ALT','110')))
    for _ in range(3):
        s.render(cam, L.FilterConfig(3.0), L.ShrinkMode.three_sigma())
