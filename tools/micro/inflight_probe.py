"""Device frames/s of the cfg-3 fly-through with 1, 2 or 3 frames in flight
(render_async over that many frame contexts; bench.py's timing)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402
import torch  # noqa: E402

tree = L.build_synthetic_tree(**bench.TREE)
cams = bench.flythrough(L)
with L.GpuScene(tree) as s:
    for c in cams[::10]:
        s.render(c, L.FilterConfig(bench.TAU_R), L.ShrinkMode.three_sigma())
    p = s.params(L.FilterConfig(bench.TAU_R), L.ShrinkMode.three_sigma(), L.RenderOptions())
    stream = torch.cuda.ExternalStream(s.stream_ptr())
    for rep in range(2):
        for n in (1, 2, 3, 4):
            s.set_inflight(n)
            for c in cams[:10]:
                s.render_async(c, p)
            s.join()
            s.sync()
            s.take_totals()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for c in cams:
                s.render_async(c, p)
            s.join()
            e1.record(stream)
            e1.synchronize()
            f, _, _ = s.take_totals()
            print(f"in flight {n}: {f / (e0.elapsed_time(e1) / 1e3):.1f} frames/s", flush=True)
