"""Benchmark: FilterGS per-frame render on the cfg-3 workload (BASELINE.json configs[2]).

Workload: synthetic 10,039,185-node LoD tree (131x131 roots, L=3, K=8, gamma 0.5,
scene seed 1, build seed 7 -- tree_builder.cpp generator), 1920x1080, a 300-frame
fly-through (keyframes descending from altitude 400 through 200 to 140, with
oblique segments; CameraPath slerp sampling, camera_path.cpp:126-180), tau_R = 3,
three-sigma extents.  A step = one frame.  value = frames/s with the tree resident in
HBM (device-timed, CUDA events on the scene stream, max over ranks); e2e = the same
frames through the reference-shaped synchronous C-ABI call lodgs_gpu_render with the
image copied back to pinned host memory every frame.

Multi-GPU (torchrun): the tree is replicated, every rank renders its own K frames of
the path (start offset rank*300/N), no collective on the data path ("weak").
--impl reference: the reference renderer itself (oracle/_ref, compiled from
/root/reference) on the host cores, bounded sample of the same path.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FPS @1080p on 10M-node LoD tree; filter+sort HBM GB/s vs peak; tile pairs"
TREE = dict(nx=131, ny=131, seed=1, depth=3, build_seed=7)
W, H, FOCAL, TAU_R = 1920, 1080, 1000.0, 3.0
PATH_SAMPLES = (100, 100, 99)  # 300 frames = sum + 1


def _normalize(v):
    return v / np.linalg.norm(v)


def look_at(eye, target, up=(0.0, 1.0, 0.0)):
    """World->camera rotation rows (x right, y down, z forward) and translation."""
    eye = np.asarray(eye, np.float64)
    f = _normalize(np.asarray(target, np.float64) - eye)
    x = _normalize(np.cross(f, np.asarray(up, np.float64)))
    y = np.cross(f, x)
    R = np.stack([x, y, f])
    t = -R @ eye
    return tuple(R.reshape(-1)), tuple(t)


def flythrough(L):
    """cfg 3 camera path: 4 keyframes, 300 frames."""
    keys = []
    for eye, target in (((0.0, 0.0, 400.0), (0.0, 0.0001, 0.0)),
                        ((30.0, -60.0, 260.0), (10.0, 10.0, 0.0)),
                        ((-20.0, 10.0, 200.0), (-20.0, 10.0001, 0.0)),
                        ((40.0, -30.0, 140.0), (50.0, 40.0, 0.0))):
        R, t = look_at(eye, target)
        keys.append(L.Camera(W, H, FOCAL, FOCAL, W / 2.0, H / 2.0, R, t, 0.01, 1000.0))
    return L.sample_camera_path(keys, PATH_SAMPLES)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def filter_traffic_bytes():
    """DRAM bytes (read + write) of the four filter kernels for one altitude-200
    frame, from the committed ncu --set full summary (tools/ncu_summary.py)."""
    path = os.path.join(ROOT, "profiles", "r1_ncu_filter_alt200.txt")
    try:
        tot, seen = 0.0, set()
        for line in open(path):
            f = line.split()
            if f and f[0] in ("k_mark_internal", "k_select_internal", "k_filter_leaves",
                              "k_compact") and f[0] not in seen:
                seen.add(f[0])
                tot += (float(f[2]) + float(f[3])) * 1e6
        return (tot if len(seen) == 4 else None), os.path.relpath(path, ROOT)
    except OSError:
        return None, None


def ncu_kernel_row(kernel, fname="r1_ncu_render_alt200.txt"):
    """One kernel's row of a committed ncu --set full summary (tools/ncu_summary.py)."""
    path = os.path.join(ROOT, "profiles", fname)
    try:
        lines = open(path).read().splitlines()
        hdr = next(ln.split() for ln in lines if ln.startswith("kernel"))
        for ln in lines:
            f = ln.split()
            if f and f[0] == kernel:
                return {h: float(v) for h, v in zip(hdr[1:], f[1:])}, os.path.relpath(path, ROOT)
    except (OSError, StopIteration, ValueError):
        pass
    return None, None


def blend_evidence():
    """The dominant kernel is issue-bound (no dense contraction, no HBM roofline):
    its SM issue utilisation from the committed ncu capture (altitude 200)."""
    for kern in ("k_blend_wsp", "k_blend_ws"):  # persistent kernel (default build) first
        row, src = ncu_kernel_row(kern)
        if row:
            break
    if not row:
        return None
    return {"kernel": kern, "bound": "issue", "issue_slots_busy_pct": row.get("issue%"),
            "sm_throughput_pct": row.get("sm%"), "achieved_occupancy_pct": row.get("occ%"),
            "ncu_us_alt200": row.get("us"), "source": src}


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_reference_sample(L, tree, cams, threads, budget_s=20.0, max_frames=6, extras=False):
    """The reference renderer (oracle/_ref) on host cores over a bounded, evenly
    strided sample of the path. FPS = frames / sum(T_total) as bench.cpp:160."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import Ref

    ref = Ref()
    h = ref.tree_from(tree)
    stride = max(1, len(cams) // max_frames)
    sample = cams[::stride][:max_frames]
    total_ms, wall, frames = 0.0, 0.0, 0
    t_start = time.perf_counter()
    for cam in sample:
        t0 = time.perf_counter()
        r = ref.render(h, cam, TAU_R, L.ShrinkMode.three_sigma(), workers=threads)
        wall += time.perf_counter() - t0
        total_ms += r["total_ms"]
        frames += 1
        if time.perf_counter() - t_start > budget_s:
            break
    # SURVEY 8(d)'s companion figures on two of the same frames: one thread, and
    # collect_kpc=true (the reference bench always renders that way, bench.cpp:128)
    extra = {}
    if extras:
        few = sample[:: max(1, len(sample) // 2)][:2]
        for name, kw in (("same_frames_all_threads", dict(workers=threads)),
                         ("single_thread", dict(workers=1)),
                         ("collect_kpc", dict(workers=threads, collect_kpc=True))):
            ms = sum(ref.render(h, cam, TAU_R, L.ShrinkMode.three_sigma(), **kw)["total_ms"]
                     for cam in few)
            extra[name] = {"value": len(few) / (ms / 1000.0), "unit": "frames/s",
                           "cores": kw["workers"], "frames": len(few)}
    ref.free_tree(h)
    return {"value": frames / (total_ms / 1000.0), "unit": "frames/s", "cores": threads,
            "kind": "reference", "cpu_model": cpu_model(),
            "sample": f"{frames} frames of the 300-frame cfg-3 path (stride {stride}), "
                      f"lodgs::render T_total (bench.cpp:160); wall incl. per-frame "
                      f"validation {frames / wall:.3f} frames/s", **extra}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, rank, world):
    from paper_2603_23891_b200 import lodgs as L

    if rank != 0:
        return
    tree = L.build_synthetic_tree(**TREE)
    cams = flythrough(L)
    threads = os.cpu_count() or 1
    per = []
    for _ in range(args.warmup):
        pass  # the reference has no device warm-up; keep W for the contract
    sample = cpu_reference_sample(L, tree, cams, threads, budget_s=60.0, max_frames=max(3, args.steps_ref))
    val = sample["value"]
    line = {"metric": METRIC, "value": val, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / val,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, seeds 1/7)",
            "config": {"workload": "cfg3: 10,039,185-node LoD tree, 1920x1080, 300-frame fly-through, "
                                   "tau_R=3, three-sigma", "nodes": tree.node_count(),
                       "width": W, "height": H},
            "impl": "reference", "cpu_baseline": sample,
            "e2e": {"value": val, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args, rank, world, local):
    import ctypes as C

    import torch

    from paper_2603_23891_b200 import lodgs as L

    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    t_build = time.perf_counter()
    tree = L.build_synthetic_tree(**TREE)
    cams = flythrough(L)
    n_path = len(cams)
    scene = L.GpuScene(tree, local)
    build_s = time.perf_counter() - t_build
    stream = torch.cuda.ExternalStream(scene.stream_ptr(), device=torch.device("cuda", local))
    params = L.RenderParamsC(TAU_R, 0.0, 0, 0)
    from paper_2603_23891_b200.sharding import reduce_timing, rotated_frames

    order = [cams[i] for i in rotated_frames(n_path, rank, world, args.warmup + args.steps)]

    # size the pair buffer on the whole path once (untimed)
    for cam in cams[:: max(1, n_path // 30)]:
        launches_per_frame = scene.render(cam, L.FilterConfig(TAU_R),
                                          L.ShrinkMode.three_sigma()).stats.kernel_launches

    def device_loop(frames, profile=False):
        scene.take_totals()
        if profile:
            scene.profile(True)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ev0.record(stream)
        for cam in frames:
            scene.render_async(cam, params)
        scene.join()  # frames alternate over two in-flight contexts
        ev1.record(stream)
        ev1.synchronize()
        ms = ev0.elapsed_time(ev1)
        tot = scene.take_totals(sort_bytes=True)
        prof = scene.profile_read() if profile else None
        if profile:
            scene.profile(False)
        return ms, tot, prof

    for cam in order[: args.warmup]:
        scene.render_async(cam, params)
    scene.sync()
    timed = order[args.warmup:]
    with ClockSampler(local) as clocks:
        for attempt in range(3):
            try:
                ms, (nf, sum_sel, sum_pairs, sum_sort_bytes), _ = device_loop(timed)
                break
            except L.InternalError:
                continue  # pair buffer grew; re-run the timed region
    # per-stage device times over a second pass of the same frames (events between kernels)
    _, _, (pf, stage_ms) = device_loop(timed, profile=True)

    # e2e through the public C ABI with host buffers: every frame's camera goes in and its
    # full f32 RGB image comes back to pinned host memory.  Default: the pipelined
    # lodgs_gpu_render_batch (frame i+1 computes while frame i copies out; a ring of
    # 4 host images); --e2e-sync: one synchronous lodgs_gpu_render call per frame.
    img_bytes = W * H * 3 * 4
    ring = []
    for _ in range(4):
        p = C.c_void_p()
        L._check(L.load_library().lodgs_gpu_host_alloc(img_bytes, C.byref(p)))
        ring.append(p.value)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e2e_frames = timed if args.e2e_steps <= 0 else timed[: max(1, min(len(timed), args.e2e_steps))]
    # untimed warm-up of both e2e legs (W frames each: first-call host allocations and
    # module loading stay out of the timed region, as for the device loop)
    warm = order[: max(1, args.warmup)]
    for rgb8 in (False, True):
        scene.render_batch(warm, L.FilterConfig(TAU_R), L.ShrinkMode.three_sigma(),
                           L.RenderOptions(output_rgb8=rgb8),
                           host_ptrs=[ring[i % 4] for i in range(len(warm))])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if args.e2e_sync:
        st = L.RenderStatsC()
        for i, cam in enumerate(e2e_frames):
            c = cam.to_c()
            L._check(L.load_library().lodgs_gpu_render(scene.handle, C.byref(c), C.byref(params),
                                                       ring[i % 4], C.byref(st)))
    else:
        scene.render_batch(e2e_frames, L.FilterConfig(TAU_R), L.ShrinkMode.three_sigma(),
                           host_ptrs=[ring[i % 4] for i in range(len(e2e_frames))])
    e2e_s = time.perf_counter() - t0
    # the same frames with 8-bit images out (the reference CLI's render -> save_ppm
    # bytes; LODGS_RENDER_OUTPUT_RGB8): 6.2 MB per 1080p frame instead of 24.9 MB
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    scene.render_batch(e2e_frames, L.FilterConfig(TAU_R), L.ShrinkMode.three_sigma(),
                       L.RenderOptions(output_rgb8=True),
                       host_ptrs=[ring[i % 4] for i in range(len(e2e_frames))])
    e2e8_s = time.perf_counter() - t0
    for p in ring:
        L.load_library().lodgs_gpu_host_free(p)

    # max over ranks of the timed regions; per-rank counters summed
    ms_max, _ = reduce_timing(dist, ms, [], device="cuda")
    e2e8_max, _ = reduce_timing(dist, e2e8_s, [], device="cuda")
    e2e_max, (sum_sel_all, sum_pairs_all, nf_all) = reduce_timing(
        dist, e2e_s, [sum_sel, sum_pairs, nf], device="cuda")
    sum_sel, sum_pairs, nf = sum_sel_all, sum_pairs_all, int(nf_all)
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    K = len(timed)
    fps = world * K / (ms_max / 1000.0)
    e2e_fps = world * len(e2e_frames) / e2e_max
    peak, peak_kind = measured_peak_gbs()
    n = tree.node_count()
    n_int = int(tree.level_offsets[-1])  # internal nodes precede the leaf level
    mean_sel = sum_sel / max(1, nf)
    mean_pairs = sum_pairs / max(1, nf)
    # B_f = 29 N + 16 N_int + 4 N_sel per frame (mark + select)
    filt_bytes = 29 * n + 16 * n_int + 4 * mean_sel
    filt_ms = (stage_ms[0] + stage_ms[1]) / max(1, pf)
    mark_ms = stage_ms[0] / max(1, pf)
    sort_ms = stage_ms[3] / max(1, pf)
    # the reference LSD radix's bytes, (24 x non-uniform 8-bit digits
    # + 8) per pair, counted per frame on the device from the frame's keys
    sort_bytes = sum_sort_bytes / max(1, nf)
    stage_names = ["filter_internal", "filter_leaves_compact", "preprocess_keys", "tile_sort", "blend"]
    per_stage = {k: round(stage_ms[i] / max(1, pf), 5) for i, k in enumerate(stage_names)}
    dominant = max(range(5), key=lambda i: stage_ms[i])
    filt_gbs = filt_bytes / (filt_ms * 1e-3) / 1e9
    traffic, traffic_src = filter_traffic_bytes()
    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_max / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, seeds 1/7; tree resident in HBM)",
        "config": {"workload": "cfg3: 10,039,185-node LoD tree, 1920x1080, 300-frame fly-through, "
                               "tau_R=3, three-sigma", "nodes": n, "width": W, "height": H,
                   "frames_per_rank": K, "l2": "inputs larger than L2 (tree 1.1 GB in HBM, "
                   "filter streams 0.3 GB per frame)", "parallelism": f"view-sharded x{world}"},
        "mean_selected": mean_sel, "mean_pairs": mean_pairs,
        "stage_ms_per_frame": per_stage,
        "roofline": {"kernel": "filter (k_mark_internal + k_select_internal + "
                                "k_filter_leaves + k_compact)", "bound": "hbm",
                     "achieved": filt_gbs, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": filt_gbs / peak, "traffic": traffic,
                     "traffic_source": f"ncu --set full dram__bytes_read+write, one altitude-200 "
                                       f"frame ({traffic_src}); the leaf pass never fetches leaves "
                                       f"under blocked parents, so traffic < algorithmic bytes",
                     "algorithmic_bytes_per_frame": filt_bytes,
                     "dominant_stage": stage_names[dominant]},
        "sort": {"kernel": "k_tile_sort + k_tile_sort_big (per-tile register bitonic on "
                           "(depth, slot) after the counting tile digit)", "bound": "hbm",
                 "achieved_gbs": sort_bytes / (sort_ms * 1e-3) / 1e9 if sort_ms > 0 else None,
                 "frac": (sort_bytes / (sort_ms * 1e-3) / 1e9) / peak if sort_ms > 0 else None,
                 "peak_gbs": peak, "algorithmic_bytes_per_frame": sort_bytes,
                 "bytes_definition": "SURVEY 8(d): (24 B x non-uniform 8-bit digits of the "
                                     "reference key tile<<32|depth + 8 B) per pair",
                 "device_traffic_per_frame": 16 * mean_pairs},
        "blend": blend_evidence(),
        "e2e": {"value": e2e_fps, "unit": "frames/s",
                "h2d_bytes_per_step": C.sizeof(L.CameraC) + C.sizeof(L.RenderParamsC),
                "d2h_bytes_per_step": img_bytes + 64, "frames": len(e2e_frames),
                "call": "lodgs_gpu_render" if args.e2e_sync else "lodgs_gpu_render_batch",
                "pcie_note": "f32 RGB image per frame (lodgs::render's Image): D2H-bound "
                             "(~56 GB/s measured, tools/micro/d2h_bw.py)"},
        "e2e_rgb8": {"value": world * len(e2e_frames) / e2e8_max, "unit": "frames/s",
                     "h2d_bytes_per_step": C.sizeof(L.CameraC) + C.sizeof(L.RenderParamsC),
                     "d2h_bytes_per_step": W * H * 3 + 64,
                     "call": "lodgs_gpu_render_batch + LODGS_RENDER_OUTPUT_RGB8 (save_ppm bytes)"},
        "gpu_launches": int(launches_per_frame) * K,
        "clocks": clocks.summary(),
        "setup_s": build_s,
    }
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_reference_sample(L, tree, cams, os.cpu_count() or 1,
                                                    budget_s=args.cpu_budget, extras=True)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=0, help="frames for e2e (0 = all timed frames)")
    ap.add_argument("--steps-ref", type=int, default=6)
    ap.add_argument("--cpu-budget", type=float, default=25.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-sync", action="store_true",
                    help="e2e through one synchronous lodgs_gpu_render per frame")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world, local)


if __name__ == "__main__":
    main()
