"""Secondary BASELINE.json workloads (the headline cfg 3 is bench.py's default).

  cfg2: 1,007,370-node tree (41x42 roots, L=3), 1920x1080, top-down altitude 50,
        GTC shrinking on (adaptive tau from GPU calibration, lambda_G given).  SH degree
        0: the reference is SH0-only, so SH3 colours would be parity-unpinned.
  cfg4: 50,142,872-node tree (103x104 roots, L=4), 3840x2160, fx=2000, a descent from
        altitude 400 to 110; GTC shrink off (three-sigma) vs on (adaptive).

Device-timed FPS (CUDA events on the scene stream), pairs per frame, the calibrated tau.
Prints one JSON object per (workload, shrink mode).

    python tools/workloads.py --which cfg2 cfg4 --frames 30
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402


def path(width, height, focal, keys, samples):
    cams = []
    for eye, target in keys:
        R, t = bench.look_at(eye, target)
        cams.append(L.Camera(width, height, focal, focal, width / 2.0, height / 2.0, R, t))
    return L.sample_camera_path(cams, samples)


def time_frames(scene, cams, mode, tau_r=3.0, reps=1):
    import torch

    stream = torch.cuda.ExternalStream(scene.stream_ptr())
    p = scene.params(L.FilterConfig(tau_r), mode, L.RenderOptions())
    for cam in cams[:3]:  # warm-up and pair-buffer sizing
        scene.render(cam, L.FilterConfig(tau_r), mode)
    for cam in cams:
        scene.render(cam, L.FilterConfig(tau_r), mode)
    scene.take_totals()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(reps):
        for cam in cams:
            scene.render_async(cam, p)
    ev1.record(stream)
    ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    frames, sel, pairs = scene.take_totals()
    return {"fps": frames / (ms / 1e3), "ms_per_frame": ms / frames, "frames": frames,
            "mean_selected": sel / frames, "mean_pairs": pairs / frames}


def run(which, frames, lambda_g):
    out = []
    if which == "cfg2":
        t0 = time.perf_counter()
        tree = L.build_synthetic_tree(nx=41, ny=42, seed=1, depth=3, build_seed=7)
        cams = path(1920, 1080, 1000.0, [((0.0, 0.0, 60.0), (0.0, 0.0001, 0.0)),
                                         ((5.0, -3.0, 50.0), (5.0, -2.9999, 0.0))],
                    [max(1, frames - 1)])
    else:
        t0 = time.perf_counter()
        tree = L.build_synthetic_tree(nx=103, ny=104, seed=1, depth=4, build_seed=7)
        n = max(2, frames) - 1
        cams = path(3840, 2160, 2000.0, [((0.0, 0.0, 400.0), (0.0, 0.0001, 0.0)),
                                         ((20.0, -10.0, 300.0), (20.0, -9.9999, 0.0)),
                                         ((-10.0, 15.0, 110.0), (-10.0, 15.0001, 0.0))],
                    [n // 2, n - n // 2])
    build_s = time.perf_counter() - t0
    with L.GpuScene(tree) as scene:
        views = cams[:: max(1, len(cams) // 4)][:4]
        rep = scene.calibrate(views, lambda_g, L.FilterConfig(3.0))
        base = {"workload": which, "nodes": tree.node_count(), "width": cams[0].width,
                "height": cams[0].height, "frames": len(cams), "tau_r": 3.0,
                "build_s": build_s, "device_bytes": scene.memory_bytes()}
        modes = [("three_sigma", L.ShrinkMode.three_sigma()),
                 ("adaptive", L.ShrinkMode.adaptive(rep.tau))]
        for name, mode in modes:
            r = time_frames(scene, cams, mode)
            rec = dict(base, shrink=name, **r)
            if name == "adaptive":
                rec.update(lambda_g=lambda_g, tau=rep.tau, calib_views=rep.n_views,
                           scene_gtc=rep.scene_mean)
            out.append(rec)
            print(json.dumps(rec), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", nargs="+", default=["cfg2", "cfg4"])
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--lambda-g", type=float, default=0.2)
    args = ap.parse_args()
    for w in args.which:
        run(w, args.frames, args.lambda_g)


if __name__ == "__main__":
    main()
