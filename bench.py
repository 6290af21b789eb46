"""Benchmark: FilterGS per-frame render on the cfg-3 workload (BASELINE.json configs[2]).

Workload: synthetic 10,039,185-node LoD tree (131x131 roots, L=3, K=8, gamma 0.5,
scene seed 1, build seed 7 -- tree_builder.cpp generator), 1920x1080, a 300-frame
fly-through (keyframes descending from altitude 400 through 200 to 140, with
oblique segments; CameraPath slerp sampling, camera_path.cpp:126-180), tau_R = 3,
three-sigma extents.  A step = one frame.

Timed frames: for any --steps K the N*K frames of the job are spread evenly over the
whole 300-frame path (frame floor(j*300/(N*K))) and dealt round-robin to the ranks
(paper_2603_23891_b200/sharding.py: strided_frames), so the timed workload is the
fly-through, not its first frames, and every rank gets the same altitude mix.

value  = frames/s with the tree resident in HBM (device-timed, CUDA events on the
         scene's control stream, max over ranks).
e2e    = the same frames through the public C ABI with host buffers: camera in, f32
         RGB image (lodgs::render's Image) out to pinned host memory every frame, via
         the pipelined lodgs_gpu_render_batch; e2e_sync does one synchronous
         lodgs_gpu_render per frame (the drop-in lodgs::render shim's call);
         e2e_rgb8 returns the 8-bit image the reference CLI writes.

Multi-GPU (torchrun): the tree is replicated, frames are sharded round-robin, no
collective on the data path ("weak": K frames per rank).

--impl reference: the reference renderer itself (oracle/_ref, compiled from
/root/reference's sources) on all host cores, on the SAME frames: tree built by the
reference's own generator (build_tree), cameras by its own CameraPath::sample, FPS =
frames / sum of RenderStats::total_ms (bench.cpp:160).  It never loads the product
library.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2603_23891_b200.sharding import reduce_timing, strided_frames  # noqa: E402

METRIC = "FPS @1080p on 10M-node LoD tree; filter+sort HBM GB/s vs peak; tile pairs"
TREE = dict(nx=131, ny=131, seed=1, depth=3, build_seed=7)
W, H, FOCAL, TAU_R = 1920, 1080, 1000.0, 3.0
VIEWS_INFLIGHT = 12  # render_views_async: three sets of four contexts, groups of four views
PATH_SAMPLES = (100, 100, 99)  # 300 frames = sum + 1
N_PATH = sum(PATH_SAMPLES) + 1
WORKLOAD = ("cfg3: 10,039,185-node LoD tree, 1920x1080, 300-frame fly-through "
            "(timed frames strided over the whole path), tau_R=3, three-sigma")
DTYPE = "f64+f32"
DTYPE_NOTE = ("filter decisions, projection, shrink radii, binning and sort keys in FP64/integer "
              "(bit-exact with the reference); blend in FP32 with a certified FP64 re-check of "
              "uncertain alpha>=1/255 decisions (image within max-abs 1e-3, north_star)")
# ncu capture of the bench's own frames (tools/ncu_frames.py): per-kernel mean time and
# DRAM bytes per launch
NCU_FRAMES = os.path.join(ROOT, "profiles", "r2_ncu_bench_frames.json")


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


def keyframes(L):
    """cfg 3 keyframes: top-down at 400, oblique at 260, top-down at 200, oblique at 140."""
    keys = []
    for eye, target in (((0.0, 0.0, 400.0), (0.0, 0.0001, 0.0)),
                        ((30.0, -60.0, 260.0), (10.0, 10.0, 0.0)),
                        ((-20.0, 10.0, 200.0), (-20.0, 10.0001, 0.0)),
                        ((40.0, -30.0, 140.0), (50.0, 40.0, 0.0))):
        R, t = look_at(eye, target)
        keys.append(L.Camera(W, H, FOCAL, FOCAL, W / 2.0, H / 2.0, R, t, 0.01, 1000.0))
    return keys


def flythrough(L):
    """cfg 3 camera path: 4 keyframes, 300 frames (the product's CameraPath::sample)."""
    return L.sample_camera_path(keyframes(L), PATH_SAMPLES)


def config(world, k):
    return {"workload": WORKLOAD, "nodes": 10039185, "width": W, "height": H,
            "frames_per_rank": k, "frame_schedule": "strided_frames(300, rank, N, K)",
            "enqueue": "render_views_async: the LoD filter shared by each group of 4 frames, "
                       "groups rotating over three sets of 4 in-flight contexts",
            "l2": "inputs larger than L2 (tree 1.1 GB in HBM, the filter streams ~0.3 GB "
                  "per frame)", "parallelism": f"view-sharded x{world}"}


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
            self._stop.wait(0.05)

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


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_frames():
    """Per-kernel mean device time (us) and DRAM MB read/written per launch over the
    bench's own timed frames (profiles/r2_ncu_bench_frames.json, tools/ncu_frames.py).
    ncu replays every launch with cold caches and serialised, so only the kernels'
    DRAM bytes and their shares of the frame are used from it, not absolute times."""
    try:
        with open(NCU_FRAMES) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


STAGE_KERNELS = {
    "filter": ("k_mark_internal", "k_select_internal", "k_filter_leaves", "k_compact"),
    "preprocess": ("k_preprocess",),
    "keys": ("k_tile_offsets_cluster", "k_tile_offsets", "k_emit_keys"),
    "sort": ("k_tile_sort", "k_tile_sort_big"),
    "blend": ("k_blend_wsp", "k_blend_tma", "k_blend_ws", "k_blend_cpa", "k_blend_g4"),
}


def stage_traffic(prof, stage):
    """DRAM bytes (read + write) per frame of a stage's kernels, from the ncu capture of
    the bench frames; None without a capture."""
    if not prof:
        return None
    ks = prof.get("kernels", {})
    tot, seen = 0.0, False
    for k in STAGE_KERNELS[stage]:
        if k in ks:
            seen = True
            tot += (ks[k]["dram_rd_mb"] + ks[k]["dram_wr_mb"]) * 1e6 * ks[k]["launches_per_frame"]
    return tot if seen else None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _ref():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import Ref

    return Ref()


def cpu_reference_sample(L, ref, h, cams, threads, frames, extras=False):
    """The reference renderer (oracle/_ref) on host cores over `frames` (indices into
    the path).  FPS = frames / sum(T_total) as bench.cpp:160."""
    total_ms, wall, pairs = 0.0, 0.0, 0
    for i in frames:
        t0 = time.perf_counter()
        r = ref.render(h, cams[i], TAU_R, L.ShrinkMode.three_sigma(), workers=threads)
        wall += time.perf_counter() - t0
        total_ms += r["total_ms"]
        pairs += r["n_pairs"]
    n = len(frames)
    out = {"value": n / (total_ms / 1000.0), "unit": "frames/s", "cores": threads,
           "kind": "reference", "cpu_model": cpu_model(), "frames": n,
           "mean_pairs": pairs / max(1, n), "wall_value": n / wall,
           "sample": f"{n} frames of the 300-frame cfg-3 path (indices {frames[0]}..{frames[-1]}, "
                     f"stride {frames[1] - frames[0] if n > 1 else 0}), lodgs::render "
                     f"T_total (bench.cpp:160); wall incl. the per-frame require_valid "
                     f"{n / wall:.3f} frames/s"}
    if extras:
        # SURVEY 8(d)'s companion figures on two of the same frames: one thread, and
        # collect_kpc=true (the reference bench always renders that way, bench.cpp:128)
        few = [frames[len(frames) // 3], frames[(2 * len(frames)) // 3]]
        for name, kw in (("same_frames_all_threads", dict(workers=threads)),
                         ("single_thread", dict(workers=1)),
                         ("collect_kpc", dict(workers=threads, collect_kpc=True))):
            ms = sum(ref.render(h, cams[i], TAU_R, L.ShrinkMode.three_sigma(), **kw)["total_ms"]
                     for i in few)
            out[name] = {"value": len(few) / (ms / 1000.0), "unit": "frames/s",
                         "cores": kw["workers"], "frames": few}
    return out


def run_reference(args, rank, world):
    """The reference arm: the unmodified reference renderer on the box's host cores,
    on this arm's config (same tree, same 300-frame path, the same strided frames).
    Rank 0 only (a CPU arm has nothing to shard over GPUs)."""
    from paper_2603_23891_b200 import lodgs as L  # data classes only: no library load

    if rank != 0:
        return
    t0 = time.perf_counter()
    ref = _ref()
    h = ref.lib.ref_build_synthetic(TREE["nx"], TREE["ny"], 2.0, 0.2, 0.6, 0.3, 0.9,
                                    TREE["seed"], 1, TREE["depth"], 0.5, 8, TREE["build_seed"])
    if not h:
        raise RuntimeError(ref.err())
    n_nodes = int(ref.lib.ref_tree_size(h))
    cams = ref.sample_path(keyframes(L), PATH_SAMPLES)
    setup_s = time.perf_counter() - t0
    threads = os.cpu_count() or 1
    k = args.steps
    frames = strided_frames(len(cams), 0, 1, k)
    for i in strided_frames(len(cams), 0, 1, args.warmup):  # untimed warm-up frames
        ref.render(h, cams[i], TAU_R, L.ShrinkMode.three_sigma(), workers=threads)
    sample = cpu_reference_sample(L, ref, h, cams, threads, frames)
    ref.free_tree(h)
    val = sample["value"]
    cfg = config(1, k)
    cfg["nodes"] = n_nodes
    line = {"metric": METRIC, "value": val, "unit": "frames/s", "n_gpus": world,
            "steps": k, "warmup": args.warmup, "ms_per_step": 1000.0 / val,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator build_tree, seeds 1/7)",
            "config": cfg, "impl": "reference", "mean_pairs": sample["mean_pairs"],
            "cpu_baseline": sample, "setup_s": setup_s,
            "e2e": {"value": val, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args, rank, world, local):
    import ctypes as C

    import torch

    from paper_2603_23891_b200 import lodgs as L

    dist = None
    # LODGS_BENCH_DIST_BACKEND=gloo: the N>1 path on a box with fewer GPUs than ranks (the
    # GPU test runs 2 ranks on one B200; ranks share a device, counters reduce on the CPU)
    backend = os.environ.get("LODGS_BENCH_DIST_BACKEND", "nccl")
    if backend == "gloo":
        local = local % max(1, torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist

        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if backend == "gloo" else "cuda"
    torch.cuda.set_device(local)
    t_build = time.perf_counter()
    tree = L.build_synthetic_tree(**TREE)
    cams = flythrough(L)
    n_path = len(cams)
    scene = L.GpuScene(tree, local)
    build_s = time.perf_counter() - t_build
    lib = L.load_library()
    stream = torch.cuda.ExternalStream(scene.stream_ptr(), device=torch.device("cuda", local))
    params = L.RenderParamsC(TAU_R, 0.0, 0, 0)
    K = args.steps
    timed_idx = strided_frames(n_path, rank, world, K)
    warm_idx = strided_frames(n_path, rank, world, args.warmup)
    timed = [cams[i] for i in timed_idx]
    warm = [cams[i] for i in warm_idx]
    mode = L.ShrinkMode.three_sigma()

    # size the pair buffer on the whole path once (untimed)
    for cam in cams[::10]:
        launches_per_frame = scene.render(cam, L.FilterConfig(TAU_R), mode).stats.kernel_launches

    def device_loop(frames, profile=False, views=False):
        scene.take_totals()
        if profile:
            scene.profile(True)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        if views:  # the LoD filter shared by each group of four frames
            scene.render_views_async(frames, params)
        else:
            for cam in frames:
                scene.render_async(cam, params)
        scene.join()  # frames rotate over the in-flight contexts; the control stream waits
        ev1.record(stream)
        ev1.synchronize()
        ms = ev0.elapsed_time(ev1)
        tot = scene.take_totals(sort_bytes=True)
        prof = scene.profile_read() if profile else None
        if profile:
            scene.profile(False)
        return ms, tot, prof

    # The headline loop: the frames through render_views_async -- the LoD filter shared
    # by each group of four frames (one pass over the node arrays), groups
    # rotating over three sets of four in-flight contexts.  Warm-up:
    # the W warm-up frames, cycled until every one of the 12 contexts has rendered.
    scene.set_inflight(VIEWS_INFLIGHT)
    warm_all = [warm[i % len(warm)] for i in range(max(len(warm), 2 * VIEWS_INFLIGHT))]
    scene.render_views_async(warm_all, params)
    scene.sync()
    with ClockSampler(local) as clocks:
        for attempt in range(3):
            try:
                ms, (nf, sum_sel, sum_pairs, sum_sort_bytes), _ = device_loop(timed, views=True)
                break
            except L.InternalError:
                continue  # pair buffer grew; re-run the timed region
    scene.set_inflight(4)
    for cam in warm:
        scene.render_async(cam, params)
    scene.sync()
    # the same frames enqueued one by one (four in flight, a filter pass per frame)
    pms, _, _ = device_loop(timed)
    pmax, _ = reduce_timing(dist, pms, [], device=red_dev)
    per_frame_fps = world * K / (pmax / 1000.0)
    # per-stage device times over a second pass of the same frames (events between
    # kernels, one frame in flight: the stage split, not the throughput)
    _, _, (pf, stage_ms) = device_loop(timed, profile=True)

    # the TMA-staged blend kernels, same frames, same loop: evidence
    # for the kernel choice, not the headline
    variants = {}
    default_params = params
    for name, flag in (("blend_wsp", 512), ("blend_tma", 64), ("blend_gather4", 128)):
        params = L.RenderParamsC(TAU_R, 0.0, 0, flag)
        for cam in warm:
            scene.render_async(cam, params)
        scene.sync()
        vms, _, _ = device_loop(timed)
        vmax, _ = reduce_timing(dist, vms, [], device=red_dev)
        variants[name] = world * K / (vmax / 1000.0)
    params = default_params

    # ---- e2e through the public C ABI with host buffers (pinned ring of 4 images)
    img_bytes = W * H * 3 * 4
    ring = []
    for _ in range(4):
        p = C.c_void_p()
        L._check(lib.lodgs_gpu_host_alloc(img_bytes, C.byref(p)))
        ring.append(p.value)
    ptrs = [ring[i % 4] for i in range(len(timed))]
    # untimed warm-up of every leg (first-call host allocations stay out of the timing)
    for rgb8 in (False, True):
        scene.render_batch(warm, L.FilterConfig(TAU_R), mode, L.RenderOptions(output_rgb8=rgb8),
                           host_ptrs=ptrs[: len(warm)])
    st = L.RenderStatsC()
    for i, cam in enumerate(warm):
        c = cam.to_c()
        L._check(lib.lodgs_gpu_render(scene.handle, C.byref(c), C.byref(params), ring[i % 4],
                                      C.byref(st)))

    def timed_host(fn):
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    e2e_s = timed_host(lambda: scene.render_batch(timed, L.FilterConfig(TAU_R), mode,
                                                  host_ptrs=ptrs))

    def sync_leg():
        for i, cam in enumerate(timed):
            c = cam.to_c()
            L._check(lib.lodgs_gpu_render(scene.handle, C.byref(c), C.byref(params),
                                          ring[i % 4], C.byref(st)))

    e2e_sync_s = timed_host(sync_leg)
    e2e8_s = timed_host(lambda: scene.render_batch(
        timed, L.FilterConfig(TAU_R), mode, L.RenderOptions(output_rgb8=True), host_ptrs=ptrs))
    for p in ring:
        lib.lodgs_gpu_host_free(p)

    # max over ranks of the timed regions; per-rank counters summed
    ms_max, _ = reduce_timing(dist, ms, [], device=red_dev)
    e2e_max, _ = reduce_timing(dist, e2e_s, [], device=red_dev)
    e2e_sync_max, _ = reduce_timing(dist, e2e_sync_s, [], device=red_dev)
    e2e8_max, (sum_sel, sum_pairs, nf, sum_sort_bytes) = reduce_timing(
        dist, e2e8_s, [sum_sel, sum_pairs, nf, sum_sort_bytes], device=red_dev)
    nf = int(nf)
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    fps = world * K / (ms_max / 1000.0)
    peak, peak_kind = measured_peak_gbs()
    n = tree.node_count()
    n_int = int(tree.level_offsets[-1])  # internal nodes precede the leaf level
    mean_sel = sum_sel / max(1, nf)
    mean_pairs = sum_pairs / max(1, nf)
    stage_names = ["filter_internal", "filter_leaves_compact", "preprocess_keys", "tile_sort",
                   "blend"]
    per_stage = {k: stage_ms[i] / max(1, pf) for i, k in enumerate(stage_names)}
    dominant = max(per_stage, key=per_stage.get)
    prof = ncu_frames()

    # SURVEY.md 8(d) algorithmic bytes per frame (reference layout) per stage
    filt_bytes = 29 * n + 16 * n_int + 4 * mean_sel
    filt_ms = per_stage["filter_internal"] + per_stage["filter_leaves_compact"]
    sort_ms = per_stage["tile_sort"]
    sort_bytes = sum_sort_bytes / max(1, nf)  # (24 x non-uniform digits + 8) B per pair

    def stage_obj(name, alg_bytes, ms, bound, note=None):
        traffic = stage_traffic(prof, name)
        o = {"bound": bound, "ms_per_frame": ms, "algorithmic_bytes": alg_bytes,
             "achieved_gbs": alg_bytes / (ms * 1e-3) / 1e9 if ms > 0 else None,
             "frac": alg_bytes / (ms * 1e-3) / 1e9 / peak if ms > 0 else None,
             "traffic": traffic,
             "physical_gbs": traffic / (ms * 1e-3) / 1e9 if traffic and ms > 0 else None,
             "physical_frac": traffic / (ms * 1e-3) / 1e9 / peak if traffic and ms > 0 else None}
        if note:
            o["note"] = note
        return o

    # preprocess and key emission share one event-timed stage; split it by the kernels'
    # shares in the ncu launch list of the same frames
    pk_ms = per_stage["preprocess_keys"]
    share_pre = 0.7
    if prof:
        ks = prof.get("kernels", {})
        t_pre = sum(ks[k]["mean_us"] * ks[k]["launches_per_frame"]
                    for k in STAGE_KERNELS["preprocess"] if k in ks)
        t_keys = sum(ks[k]["mean_us"] * ks[k]["launches_per_frame"]
                     for k in STAGE_KERNELS["keys"] if k in ks)
        if t_pre + t_keys > 0:
            share_pre = t_pre / (t_pre + t_keys)
    # mean projected gaussians ~ selected (near-plane drops are rare on this path)
    stages = {
        "filter": stage_obj("filter", filt_bytes, filt_ms, "hbm",
                            "B_f = 29 N + 16 N_int + 4 N_sel; the device skips leaves under "
                            "blocked parents, so traffic < B_f"),
        "preprocess": stage_obj("preprocess", 60 * mean_sel + 52 * mean_sel, pk_ms * share_pre,
                                "hbm+fp64", "60 N_sel read + 52 N_g written (8(d)); split from "
                                "preprocess_keys by the ncu time shares"),
        "keys": stage_obj("keys", 16 * mean_sel + 12 * mean_pairs, pk_ms * (1 - share_pre),
                          "l2 atomics", "16 N_g + 12 N_P (8(d))"),
        "sort": stage_obj("sort", sort_bytes, sort_ms, "issue",
                          "reference LSD-radix bytes (24 B x non-uniform 8-bit digits + 8 B per "
                          "pair); the device sorts per tile in registers and moves 16 B/pair: "
                          "issue-bound, not HBM-bound"),
    }
    filt = stages["filter"]
    roofline = {"kernel": "filter (k_mark_internal + k_select_internal + k_filter_leaves + "
                          "k_compact)", "bound": "hbm", "achieved": filt["achieved_gbs"],
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": filt["frac"],
                "traffic": filt["traffic"], "physical_frac": filt["physical_frac"],
                "traffic_source": (f"ncu dram__bytes_read+write over the bench's own frames "
                                   f"({os.path.relpath(NCU_FRAMES, ROOT)})" if prof else None),
                "algorithmic_bytes_per_frame": filt_bytes, "dominant_stage": dominant}
    blend = {"kernel": "k_blend_cpa", "bound": "issue", "ms_per_frame": per_stage["blend"],
             "share_of_frame": per_stage["blend"] / max(1e-9, sum(per_stage.values()))}
    if prof and "k_blend_cpa" in prof.get("kernels", {}):
        kb = prof["kernels"]["k_blend_cpa"]
        blend.update({k: kb[k] for k in ("issue_pct", "sm_pct", "occ_pct") if k in kb})
    e2e_h2d = C.sizeof(L.CameraC) + C.sizeof(L.RenderParamsC)
    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_max / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": DTYPE, "dtype_note": DTYPE_NOTE,
        "data": "synthetic (reference generator restated bit-for-bit, seeds 1/7; tree "
                "resident in HBM)",
        "config": config(world, K),
        "frames": timed_idx if world == 1 else f"{K} per rank, round-robin over the path",
        "mean_selected": mean_sel, "mean_pairs": mean_pairs,
        # north_star's secondary unit: the same throughput as selected Gaussians (LoD nodes
        # the filter keeps) and (Gaussian, tile) pairs per second
        "gaussians_per_s": fps * mean_sel, "pairs_per_s": fps * mean_pairs,
        "stage_ms_per_frame": per_stage,
        "roofline": roofline, "stages": stages, "blend": blend,
        "per_frame_fps": per_frame_fps,
        "per_frame_note": "the same frames through render_async, one filter pass per frame, "
                          "four in flight (the blend-kernel variants below are measured so)",
        "blend_kernel_variants_fps": {"blend_cpa (default)": per_frame_fps, **variants},
        "e2e": {"value": world * K / e2e_max, "unit": "frames/s",
                "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": img_bytes + 64,
                "frames": K, "call": "lodgs_gpu_render_batch (pipelined over frames in flight)",
                "pcie_note": "f32 RGB image per frame (lodgs::render's Image): D2H-bound "
                             "(~56 GB/s measured, tools/micro/d2h_bw.py)"},
        "e2e_sync": {"value": world * K / e2e_sync_max, "unit": "frames/s",
                     "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": img_bytes + 64,
                     "call": "lodgs_gpu_render, one synchronous call per frame (the drop-in "
                             "lodgs::render shim's call) into pinned host memory: blend in 4 "
                             "bands, each band's rows copied while the next blends"},
        "e2e_rgb8": {"value": world * K / e2e8_max, "unit": "frames/s",
                     "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": W * H * 3 + 64,
                     "call": "lodgs_gpu_render_batch + LODGS_RENDER_OUTPUT_RGB8 (save_ppm bytes)"},
        # per frame: the 11 kernels of a single-view frame minus its 4 filter kernels, plus
        # the 4 multi-view filter kernels once per group of four frames (cfg 3: 1,226
        # compaction tiles, no prefix kernel)
        "gpu_launches": (int(launches_per_frame) - 4) * K + 4 * ((K + 3) // 4),
        "clocks": clocks.summary(),
        "setup_s": build_s,
    }
    if world == 1 and not args.no_cpu:
        ref = _ref()
        h = ref.tree_from(tree)
        line["cpu_baseline"] = cpu_reference_sample(
            L, ref, h, cams, os.cpu_count() or 1, strided_frames(n_path, 0, 1, args.cpu_frames),
            extras=True)
        ref.free_tree(h)
    print(json.dumps(line), flush=True)
    scene.close()
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-frames", type=int, default=30,
                    help="frames of the reference CPU sample (stride 300/n over the path)")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 1 or args.steps < 1:
        ap.error("--steps and --warmup must be >= 1")
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world, local)


if __name__ == "__main__":
    main()
