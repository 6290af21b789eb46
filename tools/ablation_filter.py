"""Serial vs parallel filter on the device (the paper's Table 2 ablation,
PAPER.md:126-137, :370-377): the cfg-3 tree at several altitudes.

  parallel: filter_parallel's kernels (k_mark_internal, k_select_internal,
            k_filter_leaves, k_compact) -- device time from the render's
            stage timer (RenderStats.t_calc_ms), median of R frames.
  serial:   filter_serial -- one kernel + barrier per level; per-level device
            times (CUDA events between the level launches), median of R runs.

Prints one JSON line per altitude.  Not a benchmark of record (bench.py is).

    python tools/ablation_filter.py --alt 400 200 140 --reps 20
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import topdown_camera  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--alt", type=float, nargs="+", default=[400.0, 200.0, 140.0])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--nx", type=int, default=131)
    ap.add_argument("--depth", type=int, default=3)
    args = ap.parse_args()
    tree = L.build_synthetic_tree(nx=args.nx, ny=args.nx, seed=1, depth=args.depth, build_seed=7)
    nl = len(tree.level_offsets)
    with L.GpuScene(tree) as s:
        for alt in args.alt:
            cam = topdown_camera(1920, 1080, 1000.0, alt)
            opts = L.RenderOptions(stage_timing=True)
            par = []
            for _ in range(args.reps + 3):
                out = s.render(cam, L.FilterConfig(3.0), L.ShrinkMode.three_sigma(), opts)
                par.append(out.stats.t_calc_ms)
            ser, levels = [], []
            for _ in range(args.reps + 3):
                lm = np.zeros(nl)
                r = s.filter_serial(cam, L.FilterConfig(3.0), level_ms=lm)
                ser.append(float(lm.sum()))
                levels.append(lm)
            par, ser = par[3:], ser[3:]
            lv = np.median(np.stack(levels[3:]), axis=0)
            print(json.dumps({
                "nodes": tree.node_count(), "levels": nl, "altitude": alt,
                "n_selected": int(out.stats.n_selected),
                "parallel_ms": float(np.median(par)), "parallel_barriers": 2,
                "serial_ms": float(np.median(ser)), "serial_passes": r.passes,
                "serial_level_ms": [round(float(x), 5) for x in lv],
                "serial_equals_parallel": bool(np.array_equal(
                    r.selected, s.filter(cam, L.FilterConfig(3.0)).selected)),
            }), flush=True)


if __name__ == "__main__":
    main()
