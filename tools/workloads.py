"""Secondary BASELINE.json workloads (the headline cfg 3 is bench.py's default).

  cfg2: 1,007,370-node tree (41x42 roots, L=3), 1920x1080, top-down altitude 50,
        GTC shrinking on (adaptive tau from GPU calibration at each lambda_G given, the
        paper's 0.2 and a gentle 0.02; PSNR / SSIM against the three-sigma frames).  --sh 3
        adds SH degree-3 colours (synthetic coefficients; the reference is SH0-only,
        SPEC.md:78, so these colours are parity-unpinned; tests/test_gpu_sh.py).
  cfg4: 50,142,872-node tree (103x104 roots, L=4), 3840x2160, fx=2000, a descent from
        altitude 400 to 110; GTC shrink off (three-sigma) vs on (adaptive).
  cfg5: view-batched rendering -- the cfg 3 tree, 1024 poses sampled from the cfg 3
        fly-through keyframes, dealt round-robin to the ranks of a torchrun
        launch (one process per GPU, tree replicated, no collective on the data path;
        max-over-ranks device time).  Device views/s through render_views_async (the
        multi-view filter, groups of four views) and through one render_async per view,
        plus views/s end to end with the
        8-bit image of every view read back (render_batch with LODGS_RENDER_OUTPUT_RGB8,
        6.2 MB per view; and one synchronous lodgs_gpu_read_image_rgb8 per view).

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


BLEND = "cpa"  # --blend: the fast-blend kernel (RenderOptions.blend_kernel)
THREE_SIGMA_ONLY = False
INFLIGHT = 4  # frames in flight of the per-frame timing (run's --inflight)
SH_DEGREE = 0  # --sh: view-dependent colour of this degree (synthetic coefficients)


def time_frames(scene, cams, mode, tau_r=3.0, reps=1):
    import torch

    stream = torch.cuda.ExternalStream(scene.stream_ptr())
    p = scene.params(L.FilterConfig(tau_r), mode, L.RenderOptions(blend_kernel=BLEND))
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
    scene.join()
    ev1.record(stream)
    ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    frames, sel, pairs = scene.take_totals()
    out = {"fps": frames / (ms / 1e3), "ms_per_frame": ms / frames, "frames": frames,
           "mean_selected": sel / frames, "mean_pairs": pairs / frames}
    # the same frames through render_views_async (the multi-view filter, groups of four
    # over two sets of four contexts)
    scene.set_inflight(8)
    scene.render_views_async(cams[:16], p)
    scene.sync()
    scene.take_totals()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(reps):
        scene.render_views_async(cams, p)
    scene.join()
    ev1.record(stream)
    ev1.synchronize()
    vms = ev0.elapsed_time(ev1)
    vf, _, _ = scene.take_totals()
    scene.set_inflight(INFLIGHT)
    out["fps_views"] = vf / (vms / 1e3)
    return out


def run_cfg5(n_views=1024):
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    tree = L.build_synthetic_tree(**bench.TREE)
    n = n_views - 1
    keys_cams = bench.flythrough(L)  # 300 frames; re-sample the same keyframes to 1024
    keys = [keys_cams[0], keys_cams[100], keys_cams[200], keys_cams[-1]]
    cams = L.sample_camera_path(keys, (n // 3, n // 3, n - 2 * (n // 3)))
    assert len(cams) == n_views
    from paper_2603_23891_b200.sharding import interleaved_shard

    mine = [cams[i] for i in interleaved_shard(n_views, rank, world)]
    with L.GpuScene(tree, local) as scene:
        mode = L.ShrinkMode.three_sigma()
        for cam in mine[:: max(1, len(mine) // 16)]:
            scene.render(cam, L.FilterConfig(bench.TAU_R), mode)  # pair-buffer sizing
        p = scene.params(L.FilterConfig(bench.TAU_R), mode, L.RenderOptions())
        stream = torch.cuda.ExternalStream(scene.stream_ptr(), device=torch.device("cuda", local))
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        scene.take_totals()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ev0.record(stream)
        for cam in mine:
            scene.render_async(cam, p)
        scene.join()
        ev1.record(stream)
        ev1.synchronize()
        ms_frames = ev0.elapsed_time(ev1)
        frames, sel, pairs = scene.take_totals()
        # view-batched: the multi-view filter, groups of four views over 8 contexts
        scene.set_inflight(8)
        scene.render_views_async(mine[:16], p)  # untimed: every context renders once
        scene.sync()
        scene.take_totals()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ev0.record(stream)
        scene.render_views_async(mine, p)
        scene.join()
        ev1.record(stream)
        ev1.synchronize()
        ms = ev0.elapsed_time(ev1)
        scene.take_totals()
        scene.set_inflight(4)
        # end to end: every view's 8-bit image back to pinned host memory through
        # render_batch (pipelined over the in-flight contexts) ...
        import ctypes as C
        lib = L.load_library()
        ring = []
        for _ in range(4):
            hp = C.c_void_p()
            L._check(lib.lodgs_gpu_host_alloc(mine[0].width * mine[0].height * 3, C.byref(hp)))
            ring.append(hp.value)
        opts8 = L.RenderOptions(output_rgb8=True)
        scene.render_batch(mine[:4], L.FilterConfig(bench.TAU_R), mode, opts8,
                           host_ptrs=ring[:4])  # untimed warm-up
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        scene.render_batch(mine, L.FilterConfig(bench.TAU_R), mode, opts8,
                           host_ptrs=[ring[i % 4] for i in range(len(mine))])
        e2e_s = time.perf_counter() - t0
        # ... and one synchronous read per view (no compute/copy overlap)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for cam in mine:
            scene.render_async(cam, p)
            scene.read_image_rgb8(cam)
        sync_s = time.perf_counter() - t0
        for hp in ring:
            lib.lodgs_gpu_host_free(hp)
        t = torch.tensor([ms, e2e_s * 1e3, sync_s * 1e3, ms_frames], device="cuda")
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            rec = {"workload": "cfg5", "nodes": tree.node_count(), "views": n_views,
                   "gpus": world, "views_per_gpu": len(mine),
                   "views_per_s": n_views / (t[0].item() / 1e3),
                   "views_per_s_per_frame_filter": n_views / (t[3].item() / 1e3),
                   "e2e_rgb8_views_per_s": n_views / (t[1].item() / 1e3),
                   "e2e_rgb8_sync_views_per_s": n_views / (t[2].item() / 1e3),
                   "mean_selected": sel / max(1, frames), "mean_pairs": pairs / max(1, frames)}
            print(json.dumps(rec), flush=True)
    if dist:
        dist.destroy_process_group()


def run(which, frames, lambda_g, inflight=2):
    if which == "cfg5":
        return run_cfg5()
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
        global INFLIGHT
        INFLIGHT = inflight
        scene.set_inflight(inflight)
        if SH_DEGREE:
            # synthetic view-dependent colour (no reference: SH0-only): seeded
            # N(0, 0.1) coefficients of degree SH_DEGREE, the 3DGS features_rest layout
            k = (SH_DEGREE + 1) ** 2 - 1
            import numpy as np
            sh = np.random.default_rng(11).normal(0.0, 0.1, (tree.node_count(), k, 3))
            scene.set_sh(SH_DEGREE, sh.astype(np.float32))
        views = cams[:: max(1, len(cams) // 4)][:4]
        base = {"workload": which, "nodes": tree.node_count(), "width": cams[0].width,
                "height": cams[0].height, "frames": len(cams), "tau_r": 3.0,
                "build_s": build_s, "device_bytes": scene.memory_bytes(),
                "frames_in_flight": inflight, "sh_degree": SH_DEGREE}
        modes = [("three_sigma", L.ShrinkMode.three_sigma(), None)]
        for lg in (lambda_g if not THREE_SIGMA_ONLY else []):
            rep = scene.calibrate(views, lg, L.FilterConfig(3.0))
            modes.append(("adaptive", L.ShrinkMode.adaptive(rep.tau), (lg, rep)))
        qviews = cams[:: max(1, len(cams) // 6)][:6]
        for name, mode, cal in modes:
            r = time_frames(scene, cams, mode)
            rec = dict(base, shrink=name, blend_kernel=BLEND, **r)
            if cal:
                lg, rep = cal
                rec.update(lambda_g=lg, tau=rep.tau, calib_views=rep.n_views,
                           scene_gtc=rep.scene_mean)
                # image quality against the three-sigma frame of the same view (SURVEY
                # 8(d)'s shrink caveat: the calibrated tau culls most splats at lambda 0.2)
                ps, ss = [], []
                for cam in qviews:
                    scene.render(cam, L.FilterConfig(3.0), L.ShrinkMode.three_sigma())
                    scene.set_reference_image()
                    scene.render(cam, L.FilterConfig(3.0), mode)
                    p_, s_ = scene.compare_reference(True)
                    ps.append(p_)
                    ss.append(s_)
                rec.update(quality_views=len(qviews), psnr_vs_three_sigma_mean=sum(ps) / len(ps),
                           psnr_vs_three_sigma_min=min(ps), ssim_vs_three_sigma_mean=sum(ss) / len(ss))
            out.append(rec)
            print(json.dumps(rec), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", nargs="+", default=["cfg2", "cfg4"])
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--lambda-g", type=float, nargs="+", default=[0.2, 0.02])
    ap.add_argument("--inflight", type=int, default=4, choices=(1, 2, 3, 4))
    ap.add_argument("--blend", default="cpa", choices=("cpa", "wsp", "tma", "gather4"))
    ap.add_argument("--three-sigma-only", action="store_true")
    ap.add_argument("--sh", type=int, default=0, choices=(0, 1, 2, 3))
    args = ap.parse_args()
    global BLEND, THREE_SIGMA_ONLY, SH_DEGREE
    SH_DEGREE = args.sh
    BLEND = args.blend
    THREE_SIGMA_ONLY = args.three_sigma_only
    for w in args.which:
        run(w, args.frames, args.lambda_g, args.inflight)


if __name__ == "__main__":
    main()
