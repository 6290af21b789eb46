"""Experiment: how much would two frames in flight (two streams) gain over one?
Two GpuScenes of the cfg-3 tree (tree uploaded twice) render alternate frames of the
path on their own streams; device time from events on a third stream with fork/join."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402

tree = L.build_synthetic_tree(**bench.TREE)
cams = bench.flythrough(L)
a, b = L.GpuScene(tree), L.GpuScene(tree)
p = a.params(L.FilterConfig(bench.TAU_R), L.ShrinkMode.three_sigma(), L.RenderOptions())
for cam in cams[::10]:
    a.render(cam, L.FilterConfig(bench.TAU_R), L.ShrinkMode.three_sigma())
    b.render(cam, L.FilterConfig(bench.TAU_R), L.ShrinkMode.three_sigma())
sa = torch.cuda.ExternalStream(a.stream_ptr())
sb = torch.cuda.ExternalStream(b.stream_ptr())
ctl = torch.cuda.Stream()
for mode in ("one", "two", "one", "two"):
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(ctl)
    sa.wait_event(ev0)
    sb.wait_event(ev0)
    for i, cam in enumerate(cams):
        s = a if (mode == "one" or i % 2 == 0) else b
        s.render_async(cam, p)
    ea, eb = torch.cuda.Event(), torch.cuda.Event()
    ea.record(sa)
    eb.record(sb)
    ctl.wait_event(ea)
    ctl.wait_event(eb)
    ev1.record(ctl)
    ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    print(mode, f"{len(cams) / (ms / 1e3):.1f} FPS")
