"""Every frame of a workload path (cfg 3: the 300-frame fly-through) through the bench's enqueue
(render_views_async, the production kernels) against the reference renderer itself
(oracle/_ref, all host threads): selected and pair counts equal, image within the
north-star tolerance (max-abs 1e-3, PSNR > 60 dB).  Writes one JSON summary line.
Test infrastructure (loads oracle/_ref); a few minutes of CPU for the reference.

    python tools/full_path_parity.py --which cfg3|cfg2|cfg4|cfg5 >> profiles/r2_full_path_parity.jsonl
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import bench  # noqa: E402
from oracle_bind import Ref  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402


def workload(which):
    """(tree, cams, [(name, mode)]) of tools/workloads.py's paths; cfg 3: the bench's."""
    import workloads as W

    if which == "cfg3":
        return (L.build_synthetic_tree(**bench.TREE), bench.flythrough(L),
                [("three_sigma", L.ShrinkMode.three_sigma())])
    if which == "cfg5":  # the 1,024 poses of tools/workloads.py run_cfg5 (cfg-3 tree)
        keys_cams = bench.flythrough(L)
        keys = [keys_cams[0], keys_cams[100], keys_cams[200], keys_cams[-1]]
        n = 1023
        return (L.build_synthetic_tree(**bench.TREE),
                L.sample_camera_path(keys, (n // 3, n // 3, n - 2 * (n // 3))),
                [("three_sigma", L.ShrinkMode.three_sigma())])
    if which == "cfg2":
        tree = L.build_synthetic_tree(nx=41, ny=42, seed=1, depth=3, build_seed=7)
        cams = W.path(1920, 1080, 1000.0, [((0.0, 0.0, 60.0), (0.0, 0.0001, 0.0)),
                                           ((5.0, -3.0, 50.0), (5.0, -2.9999, 0.0))], [29])
        # the device-calibrated taus of lambda_G 0.2 / 0.02 (profiles/r2_workloads_*)
        return tree, cams, [("three_sigma", L.ShrinkMode.three_sigma()),
                            ("adaptive_0.797", L.ShrinkMode.adaptive(0.7972857536526123)),
                            ("adaptive_0.0797", L.ShrinkMode.adaptive(0.07972857536526123))]
    tree = L.build_synthetic_tree(nx=103, ny=104, seed=1, depth=4, build_seed=7)
    cams = W.path(3840, 2160, 2000.0, [((0.0, 0.0, 400.0), (0.0, 0.0001, 0.0)),
                                       ((20.0, -10.0, 300.0), (20.0, -9.9999, 0.0)),
                                       ((-10.0, 15.0, 110.0), (-10.0, 15.0001, 0.0))], [14, 15])
    return tree, cams, [("three_sigma", L.ShrinkMode.three_sigma()),
                        ("adaptive_0.0844", L.ShrinkMode.adaptive(0.08441517068141142))]


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="cfg3", choices=("cfg2", "cfg3", "cfg4", "cfg5"))
    args = ap.parse_args()
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    ref = Ref()
    threads = os.cpu_count() or 1
    tree, cams, modes = workload(args.which)
    rh = ref.tree_from(tree)
    for mname, mode in modes:
        run(ref, rh, tree, cams, mode, mname, args.which, threads)


def run(ref, rh, tree, cams, mode, mname, which, threads):
    t0 = time.perf_counter()
    with L.GpuScene(tree) as s:
        s.set_inflight(12 if which != "cfg4" else 8)
        for c in cams[::10]:
            s.render(c, L.FilterConfig(bench.TAU_R), mode)  # pair-buffer sizing
        p = s.params(L.FilterConfig(bench.TAU_R), mode, L.RenderOptions())
        worst_err, worst_psnr, bad, count_mismatch = 0.0, float("inf"), [], []
        for b in range(0, len(cams), 20):
            chunk = cams[b:b + 20]
            imgs = [np.empty((c.height, c.width, 3), np.float32) for c in chunk]
            s.take_totals()
            s.render_views_async(chunk, p, host_ptrs=[im.ctypes.data for im in imgs])
            s.sync()
            nf, gsel, gpairs = s.take_totals()
            wsel = wpairs = 0
            for k, (c, im) in enumerate(zip(chunk, imgs)):
                want = ref.render(rh, c, bench.TAU_R, mode, workers=threads)
                wsel += want["n_selected"]
                wpairs += want["n_pairs"]
                err = float(np.abs(im.astype(np.float64) - want["image"]).max())
                psnr = ref.psnr(im, want["image"]) if err > 0 else float("inf")
                worst_err = max(worst_err, err)
                worst_psnr = min(worst_psnr, psnr)
                if err > 1e-3 or psnr <= 60.0:
                    bad.append(b + k)
            if (nf, gsel, gpairs) != (len(chunk), wsel, wpairs):
                count_mismatch.append(b)
    print(json.dumps({"workload": which, "shrink": mname, "frames": len(cams),
                      "tree_nodes": tree.node_count(),
                      "enqueue": "render_views_async (groups of 4)",
                      "worst_max_abs": worst_err, "worst_psnr_db": worst_psnr,
                      "frames_out_of_tolerance": bad, "tolerance": "max-abs 1e-3, PSNR > 60 dB",
                      "chunks_with_count_mismatch": count_mismatch,
                      "counts": "selected and pair totals per 20-frame chunk equal the reference's",
                      "reference_threads": threads,
                      "wall_s": time.perf_counter() - t0}))


if __name__ == "__main__":
    main()
