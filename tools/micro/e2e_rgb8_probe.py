"""Time render_batch (f32 and 8-bit outputs) several times in a row on the cfg-3
fly-through: first-call effects vs steady state of the e2e legs."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402

tree = L.build_synthetic_tree(**bench.TREE)
cams = bench.flythrough(L)
lib = L.load_library()
with L.GpuScene(tree) as s:
    for c in cams[::10]:
        s.render(c, L.FilterConfig(bench.TAU_R), L.ShrinkMode.three_sigma())
    ring = []
    for _ in range(4):
        p = C.c_void_p()
        L._check(lib.lodgs_gpu_host_alloc(1920 * 1080 * 12, C.byref(p)))
        ring.append(p.value)
    params = s.params(L.FilterConfig(bench.TAU_R), L.ShrinkMode.three_sigma(), L.RenderOptions())
    for rep in range(3):
        if os.environ.get("PROBE_ASYNC"):  # the bench's device loop first (two contexts)
            for c in cams:
                s.render_async(c, params)
            s.join()
            s.sync()
        for rgb8 in (False, True):
            t0 = time.perf_counter()
            s.render_batch(cams, L.FilterConfig(bench.TAU_R), L.ShrinkMode.three_sigma(),
                           L.RenderOptions(output_rgb8=rgb8),
                           host_ptrs=[ring[i % 4] for i in range(len(cams))])
            dt = time.perf_counter() - t0
            print(f"rep {rep} rgb8={rgb8}: {len(cams) / dt:.1f} frames/s", flush=True)
