"""Cull / work-distribution probe for the blend, on the oracle's
BlendList of cfg-3 path frames (CPU, numpy; no GPU):

* box hits: (splat, 8x4 block) pairs whose alpha box overlaps the block (what
  k_blend_* iterate over), vs exact ellipse-vs-block hits;
* the fraction of a hit's 32 lanes inside the alpha ellipse;
* warp iterations per 32-splat chunk for alternative work splits: half / quarter
  warps with their own lists, lane-private lists (max over lanes);
* hits for larger blocks (8x8, 16x4, 16x8) relative to 8x4.

    python tools/blend_cull_probe.py --frames 100 200 280
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import bench  # noqa: E402
from oracle_bind import Oracle  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, nargs="+", default=[100, 200, 280])
    args = ap.parse_args()
    o = Oracle()
    tree = L.build_synthetic_tree(**bench.TREE)
    cams = bench.flythrough(L)
    for fi in args.frames:
        r = o.render(tree, cams[fi], 3.0, L.ShrinkMode.three_sigma(), collect_kpc=True)
        g, p = r["gaussians"], r["pairs"]
        gi = p["gaussian"].astype(np.int64)
        t = p["tile"].astype(np.int64)
        mx = g.mean_x[gi] - (t % 120) * 16.0
        my = g.mean_y[gi] - (t // 120) * 16.0
        a, b, c, op = g.conic_a[gi], g.conic_b[gi], g.conic_c[gi], g.opacity[gi]
        thr = np.log(255 * op)
        det = a * c - b * b
        hx = np.sqrt(np.maximum(2 * thr * c / det, 0))
        hy = np.sqrt(np.maximum(2 * thr * a / det, 0))
        tstart = np.searchsorted(t, t, side="left")
        chunk = (np.arange(len(p)) - tstart) // 32
        uk, inv = np.unique(t * 100000 + chunk, return_inverse=True)

        def boxhit(x0, x1, y0, y1):
            return (thr > 0) & (mx - hx <= x1) & (mx + hx >= x0) & (my - hy <= y1) & (my + hy >= y0)

        def hits(W, H):
            return sum(boxhit(bx + 0.5, bx + W - 0.5, by + 0.5, by + H - 0.5).sum()
                       for bx in range(0, 16, W) for by in range(0, 16, H))

        box = ell = useful = 0
        it_block = it_half = it_quarter = it_lane = 0.0
        for w in range(8):
            bx, by = (w & 1) * 8, (w >> 1) * 4
            hb = boxhit(bx + 0.5, bx + 7.5, by + 0.5, by + 3.5)
            box += hb.sum()
            it_block += np.bincount(inv, weights=hb, minlength=len(uk)).sum()
            hs = [np.bincount(inv, weights=boxhit(bx + qx * 4 + 0.5, bx + qx * 4 + 3.5, by + 0.5,
                                                   by + 3.5), minlength=len(uk)) for qx in (0, 1)]
            it_half += np.max(np.stack(hs), axis=0).sum()
            qs = [np.bincount(inv, weights=boxhit(bx + qx * 4 + 0.5, bx + qx * 4 + 3.5,
                                                   by + qy * 2 + 0.5, by + qy * 2 + 1.5),
                              minlength=len(uk)) for qx in (0, 1) for qy in (0, 1)]
            it_quarter += np.max(np.stack(qs), axis=0).sum()
            idx = np.flatnonzero(hb)
            px = bx + np.arange(8) + 0.5
            py = by + np.arange(4) + 0.5
            DX = px[None, :, None] - mx[idx, None, None]
            DY = py[None, None, :] - my[idx, None, None]
            E = 0.5 * (a[idx, None, None] * DX * DX + c[idx, None, None] * DY * DY) + \
                b[idx, None, None] * DX * DY
            inside = (E <= thr[idx, None, None]).reshape(len(idx), 32)
            ell += inside.any(axis=1).sum()
            useful += inside.sum()
            per = np.zeros((len(uk), 32))
            np.add.at(per, inv[idx], inside)
            it_lane += per.max(axis=1).sum()
        h84 = hits(8, 4)
        print(f"frame {fi}: pairs {len(p)} box-hits {box} ellipse-hits {ell / box:.2f} "
              f"useful-lanes {useful / (box * 32):.2f} | iterations half {it_half / it_block:.2f} "
              f"quarter {it_quarter / it_block:.2f} lane {it_lane / it_block:.2f} | hits 8x8 "
              f"{hits(8, 8) / h84:.2f} 16x4 {hits(16, 4) / h84:.2f} 16x8 {hits(16, 8) / h84:.2f}",
              flush=True)


if __name__ == "__main__":
    main()
