import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import bench
from paper_2603_23891_b200 import lodgs as L
tree = L.build_synthetic_tree(**bench.TREE)
cams = bench.flythrough(L)
frames = cams[100:120]
with L.GpuScene(tree) as s:
    p = s.params(L.FilterConfig(3.0), L.ShrinkMode.three_sigma(), L.RenderOptions())
    for c in frames[:4]:
        s.render(c, L.FilterConfig(3.0), L.ShrinkMode.three_sigma())
    import ctypes
    if sys.argv[1] == "views":
        s.render_views_async(frames, p)
    else:
        for c in frames:
            s.render_async(c, p)
    s.sync()
