"""Shared test fixtures restating the reference's test generators.

Cameras and random configurations are drawn with the oracle's mt19937_64
restatement so they equal the reference tests' draws (rng.hpp:11-33,
test_util.hpp:19-77).
"""
from __future__ import annotations

import math
import os

import numpy as np

from paper_2603_23891_b200 import lodgs as L

# acceptance.cpp:100-104 shapes (depth, children, nx, ny, congestion)
ACCEPT_SHAPES = [
    (2, 8, 3, 3, 1), (3, 8, 2, 2, 1), (4, 5, 2, 2, 1), (5, 3, 3, 2, 1),
    (6, 2, 3, 3, 2), (6, 4, 3, 3, 2), (2, 6, 4, 4, 2), (3, 4, 3, 3, 1),
    (4, 3, 2, 3, 2), (5, 4, 2, 2, 1), (6, 3, 2, 2, 1), (2, 1, 5, 5, 1),
    (3, 7, 2, 2, 1),
]


def acceptance_filter_configs(oracle):
    """Yields (tree, camera, tau_r) exactly as acceptance.cpp:93-135 draws them
    (208 configurations)."""
    rng = oracle.rng(20240801)
    for s, (depth, k, nx, ny, cong) in enumerate(ACCEPT_SHAPES):
        for rep in range(2):
            gamma = np.float32(oracle.uniform(rng, 0.3, 0.7))
            tree = L.make_tree(900 + s * 10 + rep, depth, k, float(gamma), nx, ny, cong)
            for _ in range(8):
                dist = oracle.uniform(rng, 2.0, 90.0)
                cam = oracle.orbit_camera(rng, 160, 120, dist)
                tau_r = oracle.uniform(rng, 0.5, 50.0)
                oracle.next_below(rng, 8)  # worker count draw (timing only)
                yield tree, cam, tau_r


def push_flat(lst: dict, mx, my, conic, opacity, color, radius, depth, node=0):
    """test_util.hpp:121-136."""
    for key, v in (("mean_x", mx), ("mean_y", my), ("conic_a", conic), ("conic_b", 0.0),
                   ("conic_c", conic), ("opacity", opacity), ("col_r", color[0]),
                   ("col_g", color[1]), ("col_b", color[2]), ("radius", radius),
                   ("depth", depth), ("node", node)):
        lst.setdefault(key, []).append(v)


def to_blendlist(d: dict) -> L.BlendList:
    return L.BlendList(**{k: np.asarray(d[k]) for k in
                          ("mean_x", "mean_y", "conic_a", "conic_b", "conic_c", "opacity",
                           "col_r", "col_g", "col_b", "radius", "depth", "node")})


def random_micro_scene(oracle, rng):
    """test_raster.cpp:235-260 / acceptance.cpp:255-280 random micro-scene."""
    w = 17 + int(oracle.next_below(rng, 60))
    h = 16 + int(oracle.next_below(rng, 50))
    n = 1 + int(oracle.next_below(rng, 30))
    d: dict = {}
    for i in range(n):
        ca = math.exp(oracle.uniform(rng, -4.0, 0.0))
        cc = math.exp(oracle.uniform(rng, -4.0, 0.0))
        rho = oracle.uniform(rng, -0.8, 0.8)
        mx = oracle.uniform(rng, -5.0, w + 5.0)
        my = oracle.uniform(rng, -5.0, h + 5.0)
        d.setdefault("mean_x", []).append(mx)
        d.setdefault("mean_y", []).append(my)
        d.setdefault("conic_a", []).append(ca)
        d.setdefault("conic_b", []).append(rho * math.sqrt(ca * cc))
        d.setdefault("conic_c", []).append(cc)
        d.setdefault("opacity", []).append(oracle.uniform(rng, 0.002, 0.99))
        d.setdefault("col_r", []).append(oracle.uniform(rng, 0.0, 1.0))
        d.setdefault("col_g", []).append(oracle.uniform(rng, 0.0, 1.0))
        d.setdefault("col_b", []).append(oracle.uniform(rng, 0.0, 1.0))
        d.setdefault("radius", []).append(oracle.uniform(rng, 1.0, 25.0))
        d.setdefault("depth", []).append(np.float32(oracle.uniform(rng, 0.1, 50.0)))
        d.setdefault("node", []).append(i)
    return w, h, to_blendlist(d)


def topdown_camera(width, height, focal, altitude, x=0.0, y=0.0):
    """Camera looking straight down the world -z axis from (x, y, altitude):
    rotation diag(1,-1,-1) (det +1), t = -R*eye (BASELINE.md section 2 probes)."""
    c = L.Camera(width, height, focal, focal, width / 2.0, height / 2.0,
                 (1, 0, 0, 0, -1, 0, 0, 0, -1), (-x, y, altitude), 0.01, 1000.0)
    return c


def max_abs(a, b):
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max()) if np.size(a) else 0.0


def write_ldgs(tree, path):
    """save_binary (scene_io.cpp:55-84) restated: LDGS v1 little-endian --
    magic, version 1, node count, level count, shrink factor, then the
    interleaved means / scales / quaternions, opacity, interleaved colours,
    parents, leaf flags, level offsets."""
    n = tree.node_count()
    with open(path, "wb") as f:
        f.write(b"LDGS")
        f.write(np.array([1, n, len(tree.level_offsets)], np.uint32).tobytes())
        f.write(np.float32(tree.shrink_factor).tobytes())
        for fields in ((tree.mean_x, tree.mean_y, tree.mean_z),
                       (tree.scale_x, tree.scale_y, tree.scale_z),
                       (tree.quat_w, tree.quat_x, tree.quat_y, tree.quat_z),
                       (tree.opacity,),
                       (tree.color_r, tree.color_g, tree.color_b)):
            f.write(np.stack([np.asarray(a, np.float32) for a in fields], axis=1).tobytes())
        f.write(np.asarray(tree.parent, np.uint32).tobytes())
        f.write(np.asarray(tree.leaf, np.uint8).tobytes())
        f.write(np.asarray(tree.level_offsets, np.uint32).tobytes())


REF_LDGS_TOOL = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                             "oracle", "_ref", "ref_ldgs_tool")


def ref_ldgs(*args):
    """Runs the reference's save_scene / load_scene natively (oracle/ref_ldgs_tool.cpp)."""
    import subprocess

    return subprocess.run([REF_LDGS_TOOL, *map(str, args)], capture_output=True, text=True,
                          check=True).stdout.strip()
