"""Device frames/s of the cfg-3 bench frames: per-frame enqueues vs the multi-view filter
(render_views_async), at 4 / 6 / 8 frames in flight.  Evidence for DESIGN.md; not a
bench line.   python tools/views_probe.py [--steps 100]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402
from paper_2603_23891_b200.sharding import strided_frames  # noqa: E402


def main():
    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    tree = L.build_synthetic_tree(**bench.TREE)
    cams = bench.flythrough(L)
    frames = [cams[i] for i in strided_frames(len(cams), 0, 1, args.steps)]
    out = {}
    with L.GpuScene(tree) as s:
        stream = torch.cuda.ExternalStream(s.stream_ptr())
        p = s.params(L.FilterConfig(bench.TAU_R), L.ShrinkMode.three_sigma(), L.RenderOptions())
        for inflight in tuple(int(x) for x in os.environ.get("VIEWS_INFLIGHT", "4,6,8").split(",")):
            s.set_inflight(inflight)
            for mode in ("frames", "views"):
                best = 0.0
                for _ in range(args.reps):
                    for c in frames[:10]:
                        s.render_async(c, p)
                    s.sync()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    e0.record(stream)
                    if mode == "views":
                        s.render_views_async(frames, p)
                    else:
                        for c in frames:
                            s.render_async(c, p)
                    s.join()
                    e1.record(stream)
                    e1.synchronize()
                    best = max(best, len(frames) / (e0.elapsed_time(e1) / 1e3))
                out[f"{mode}@{inflight}"] = round(best, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
