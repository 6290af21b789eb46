import os, sys, time
sys.path.insert(0, os.getcwd())
import bench
from paper_2603_23891_b200 import lodgs as L
import torch
tree = L.build_synthetic_tree(**bench.TREE)
cams = bench.flythrough(L)
frames = cams[::3][:100]
with L.GpuScene(tree) as s:
    p = s.params(L.FilterConfig(3.0), L.ShrinkMode.three_sigma(), L.RenderOptions())
    for c in frames[:10]: s.render_async(c, p)
    s.sync()
    for mode in ("frames", "views"):
        s.set_inflight(8 if mode == "views" else 4)
        s.render_views_async(frames[:16], p); s.sync()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if mode == "views":
            s.render_views_async(frames, p)
        else:
            for c in frames: s.render_async(c, p)
        t1 = time.perf_counter()
        s.sync(); torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(mode, "host enqueue us/frame", round((t1 - t0) / len(frames) * 1e6, 1), "total us/frame", round((t2 - t0) / len(frames) * 1e6, 1))
