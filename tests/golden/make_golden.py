"""Generates tests/golden/golden_v1.npz from the REFERENCE library compiled in place
(oracle/_ref/libref_lodgs.so, built from /root/reference/proj by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixture travels with the repo, so the oracle can be pinned against the
reference's own outputs where the reference is absent (the GPU box).
Hashes are SHA-256 of the raw little-endian array bytes.
"""
import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle_bind import Ref  # noqa: E402
from paper_2603_23891_b200 import lodgs as L  # noqa: E402


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def list_hash(bl) -> str:
    return hashlib.sha256(b"".join(np.ascontiguousarray(getattr(bl, f)).tobytes()
                                   for f in L._LIST_F64 + ("depth", "node"))).hexdigest()


# (seed, depth, children, gamma, nx, ny, congestion, cam_seed, w, h, dist, tau_r, shrink kind, tau)
SCENES = [
    (5, 2, 8, 0.5, 3, 3, 1, 40, 160, 120, 12.0, 6.0, 0, 0.0),
    (21, 3, 8, 0.5, 3, 3, 2, 8, 200, 150, 14.0, 4.0, 0, 0.0),
    (21, 3, 8, 0.5, 3, 3, 2, 8, 200, 150, 14.0, 4.0, 1, 1.0 / 255.0),
    (33, 3, 8, 0.5, 3, 3, 3, 5, 200, 150, 16.0, 5.0, 2, 0.1),
    (13, 2, 8, 0.5, 3, 3, 1, 77, 128, 96, 12.0, 8.0, 2, 0.3),
    (8008, 2, 8, 0.5, 4, 4, 4, 88, 160, 120, 12.0, 16.0, 0, 0.0),
]

# synthetic generator specs (nx, ny, seed, congestion, depth, gamma, children, build_seed)
TREES = [
    (3, 3, 5, 1, 2, 0.5, 8, 5 * 1099511628211 + 11),
    (2, 3, 902, 2, 4, 0.45, 3, 7),
    (37, 37, 1, 1, 2, 0.5, 8, 7),
    (4, 4, 8008, 4, 2, 0.5, 8, 8008 * 1099511628211 + 11),
]


def main():
    ref = Ref()
    out = {}
    # exp_mx on the blend range (fastexp.hpp:38-50)
    xs = np.linspace(-32.0, 0.0, 4097)
    out["exp_x"] = xs
    out["exp_y"] = np.array([ref.exp_mx(float(x)) for x in xs])
    # effective_radius (rasterizer.cpp:36-46)
    er = []
    for sigma in (0.5, 1.0, 2.0, 7.3):
        for op in (0.05, 0.25, 0.5, 0.7, 0.9, 1.0):
            for kind, tau in ((0, 0.0), (1, 1.0 / 255.0), (2, 0.1), (2, 0.25), (2, 0.6)):
                er.append((sigma, op, kind, tau, ref.effective_radius(sigma, np.float32(op), kind, tau)))
    out["eff_radius"] = np.array(er)
    # generator trees
    for i, (nx, ny, seed, cong, depth, gamma, k, bseed) in enumerate(TREES):
        hd, t = ref.build_synthetic(nx, ny, seed=seed, congestion=cong, depth=depth, shrink=gamma,
                                    children=k, build_seed=bseed & 0xFFFFFFFFFFFFFFFF)
        out[f"tree{i}_n"] = np.array([t.node_count()])
        out[f"tree{i}_hash"] = np.array([h(np.concatenate([getattr(t, f).view(np.uint8)
                                                           for f in L._FIELDS + ("parent", "leaf", "level_offsets")]))])
        ref.free_tree(hd)
    # scenes through the reference render (rasterizer.cpp:167-213)
    for i, (seed, depth, k, gamma, nx, ny, cong, cseed, w, hh, dist, tau_r, kind, tau) in enumerate(SCENES):
        hd, t = ref.make_tree(seed, depth, k, gamma, nx, ny, cong)
        rng = ref.rng(cseed)
        cam = ref.orbit_camera(rng, w, hh, dist)
        mode = L.ShrinkMode(kind, tau)
        r = ref.render(hd, cam, tau_r, mode, collect_kpc=True)
        sel, _, _ = ref.filter(hd, t.node_count(), cam, tau_r)
        out[f"scene{i}_cam"] = np.array(list(cam.to_c().rotation) + list(cam.to_c().translation) +
                                        [cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height])
        out[f"scene{i}_counts"] = np.array([r["n_selected"], r["n_pairs"], r["n_gaussians"]])
        out[f"scene{i}_hashes"] = np.array([h(sel), h(r["pairs"]), h(r["image"]), h(r["kpc"]),
                                            list_hash(r["gaussians"])])
        ref.free_tree(hd)
    # sort KAT: 100K pairs, 1000 tiles, 50 depths (test_raster.cpp:120-135)
    rng = ref.rng(99)
    n = 100000
    pairs = np.empty(n, L.PAIR_DTYPE)
    for i in range(n):
        tile = ref.lib.ref_rng_next_below(rng, 1000)
        d = ref.lib.ref_rng_next_below(rng, 50)
        pairs[i] = (tile, np.float32(d), i)
    out["sort_in_hash"] = np.array([h(pairs)])
    ref.sort_pairs(pairs)
    out["sort_out_hash"] = np.array([h(pairs)])
    # blend micro-scenes (acceptance.cpp:255-288): image hashes of the reference blend
    sys.path.insert(0, os.path.dirname(HERE))
    from oracle_bind import Oracle
    from helpers import random_micro_scene

    orc = Oracle()
    rng = orc.rng(55)
    hs = []
    for rep in range(50):
        w, hh, bl = random_micro_scene(orc, rng)
        p = ref.bin_to_tiles(bl, w, hh)
        ref.sort_pairs(p)
        hs.append(h(ref.alpha_blend(p, bl, w, hh)))
    out["micro_hashes"] = np.array(hs)
    # bench camera path (camera_path.cpp:126-180)
    import bench

    keys = []
    for eye, target in (((0.0, 0.0, 400.0), (0.0, 0.0001, 0.0)),
                        ((30.0, -60.0, 260.0), (10.0, 10.0, 0.0)),
                        ((-20.0, 10.0, 200.0), (-20.0, 10.0001, 0.0)),
                        ((40.0, -30.0, 140.0), (50.0, 40.0, 0.0))):
        R, tt = bench.look_at(eye, target)
        keys.append(L.Camera(1920, 1080, 1000.0, 1000.0, 960.0, 540.0, R, tt, 0.01, 1000.0))
    frames = ref.sample_path(keys, bench.PATH_SAMPLES)
    arr = np.array([[*f.rotation, *f.translation, f.fx, f.fy, f.cx, f.cy, f.near, f.far]
                    for f in frames])
    out["path_frames"] = arr
    np.savez_compressed(os.path.join(HERE, "golden_v1.npz"), **out)
    print("wrote", os.path.join(HERE, "golden_v1.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
