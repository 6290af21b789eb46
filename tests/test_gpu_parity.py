"""GPU parity: the sm_100a kernels (through the C ABI) against the C oracle.

Bit-exact: vis/qpass/radius marks, selected lists, BlendList FP64 fields,
per-gaussian tile counts, N_P, sorted (tile, depth, gaussian) sequences and
the exact-mode image.  Tolerance (BASELINE.json north_star): fast-mode image
max-abs <= 1e-3 per channel and PSNR > 60 dB against the oracle image.
"""
import math

import numpy as np
import pytest

from helpers import (acceptance_filter_configs, max_abs, push_flat, random_micro_scene,
                     to_blendlist, topdown_camera)

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-3   # BASELINE.json north_star: max-abs 1e-3 per channel
PSNR_MIN = 60.0  # ... and PSNR > 60 dB


# ------------------------------------------------------------------ mark --
def test_mark_bit_identical(L, oracle, gpu):
    """test_kernels.cpp:128-171: vis / qpass / radius bit-identical, ragged
    ranges, sentinels outside [begin, end) untouched."""
    rng = oracle.rng(11)
    for rep in range(12):
        tree = L.make_tree(200 + rep, 2 + rep % 3, 8, 0.5, 3, 3)
        n = tree.node_count()
        cam = oracle.orbit_camera(rng, 320, 240, oracle.uniform(rng, 2.0, 60.0))
        tau_r = oracle.uniform(rng, 0.5, 40.0)
        begin = int(oracle.next_below(rng, 5))
        end = n - int(oracle.next_below(rng, 5))
        v0, q0, r0 = oracle.mark(tree, cam, tau_r, begin, end)
        with L.GpuScene(tree) as s:
            vis = np.full(n, 9, np.uint8)
            q = np.full(n, 9, np.uint8)
            rad = np.full(n, -1.0)
            s.mark(cam, tau_r, begin, end, vis, q, rad)
        inside = slice(begin, end)
        assert np.array_equal(vis[inside], v0[inside])
        assert np.array_equal(q[inside], q0[inside])
        assert rad[inside].tobytes() == r0[inside].tobytes()
        assert (vis[:begin] == 9).all() and (vis[end:] == 9).all()
        assert (q[:begin] == 9).all() and (q[end:] == 9).all()


# ---------------------------------------------------------------- filter --
def test_filter_acceptance_208_configs(L, oracle, gpu):
    """acceptance.cpp:93-135 (#1): 208 randomized configurations, selected
    lists bit-identical to the oracle, passes = barriers = 2."""
    count = 0
    scene = None
    last_tree = None
    for tree, cam, tau_r in acceptance_filter_configs(oracle):
        if tree is not last_tree:
            if scene:
                scene.close()
            scene = L.GpuScene(tree)
            last_tree = tree
        want, _, _ = oracle.filter(tree, cam, tau_r)
        got = scene.filter(cam, L.FilterConfig(tau_r, 1))
        assert np.array_equal(got.selected, want), f"config {count}"
        assert got.passes == 2 and got.barriers == 2
        count += 1
    scene.close()
    assert count == 208


def _leaf_tree(L, mean, scale):
    n = 1
    t = L.LoDTree.empty(n, 1)
    t.mean_x[0], t.mean_y[0], t.mean_z[0] = mean
    t.scale_x[0], t.scale_y[0], t.scale_z[0] = scale
    t.quat_w[0] = 1.0
    t.opacity[0] = 0.8
    t.color_r[0], t.color_g[0], t.color_b[0] = 0.9, 0.4, 0.1
    t.parent[0] = L.ROOT_PARENT
    t.leaf[0] = 1
    return t


def _hand_tree(L, depth, children):
    """build_tree of one root at (0,0,10), unit scale, identity rotation
    (test_filter.cpp:14-24 base_node + tree_builder.cpp:94-124)."""
    means, scales, parents, leafs, offs = [(0.0, 0.0, 10.0)], [1.0], [L.ROOT_PARENT], [depth == 0], [0]
    begin, end = 0, 1
    for level in range(1, depth + 1):
        offs.append(len(means))
        for p in range(begin, end):
            for cn in range(children):
                s = scales[p]
                off = [(0.5 if cn & b else -0.5) * s for b in (1, 2, 4)]
                means.append(tuple(float(np.float32(means[p][i] + off[i])) for i in range(3)))
                scales.append(float(np.float32(s) * np.float32(0.5)))
                parents.append(p)
                leafs.append(level == depth)
        begin, end = end, len(means)
    n = len(means)
    t = L.LoDTree.empty(n, depth + 1)
    for i in range(n):
        t.mean_x[i], t.mean_y[i], t.mean_z[i] = means[i]
        t.scale_x[i] = t.scale_y[i] = t.scale_z[i] = scales[i]
        t.quat_w[i] = 1.0
        t.opacity[i] = 0.8
        t.color_r[i], t.color_g[i], t.color_b[i] = 0.9, 0.4, 0.1
        t.parent[i] = parents[i]
        t.leaf[i] = leafs[i]
    t.level_offsets[:] = offs
    return t


def test_filter_hand_kats(L, oracle, gpu):
    """test_filter.cpp:59-108: a large visible leaf is selected; a qualifying
    internal node shadows its subtree; tau_r picks the level on a 3-chain."""
    cam = oracle.front_camera(200, 200)
    t = _hand_tree(L, 0, 8)
    with L.GpuScene(t) as s:
        assert s.filter(cam, L.FilterConfig(3.0)).selected.tolist() == [0]
    t9 = _hand_tree(L, 1, 8)
    assert t9.node_count() == 9 and L.validate_tree(t9) == 0
    _, _, r = oracle.mark(t9, cam, 1e9)
    with L.GpuScene(t9) as s:
        assert s.filter(cam, L.FilterConfig(r[0] + 1.0)).selected.tolist() == [0]
    t3 = _hand_tree(L, 2, 1)
    _, _, r = oracle.mark(t3, cam, 1e9)
    assert r[2] < r[1] < r[0]
    with L.GpuScene(t3) as s:
        for tau_r, want in (((r[2] + r[1]) / 2, [2]), ((r[1] + r[0]) / 2, [1]), (r[0] + 1.0, [0])):
            assert s.filter(cam, L.FilterConfig(tau_r)).selected.tolist() == want
            assert oracle.filter(t3, cam, tau_r)[0].tolist() == want


def test_filter_empty_and_lookaway(L, oracle, gpu):
    """test_filter.cpp:200-211: a camera looking away selects nothing."""
    t = L.make_tree(3, 3, 8, 0.5, 2, 2)
    cam = oracle.front_camera(200, 200)
    cam.translation = (0, 0, -100)
    with L.GpuScene(t) as s:
        assert s.filter(cam, L.FilterConfig(3.0)).selected.size == 0
        with pytest.raises(L.ValidationError):
            s.filter(cam, L.FilterConfig(0.0))


def test_filter_10m_tree_bit_exact(L, oracle, gpu):
    """Full-size cfg 3 tree (10,039,185 nodes): selected list bit-exact at
    three altitudes of the fly-through."""
    tree = L.build_synthetic_tree(nx=131, ny=131, seed=1, depth=3, build_seed=7)
    assert tree.node_count() == 10039185
    with L.GpuScene(tree) as s:
        for alt in (400.0, 200.0, 140.0):
            cam = topdown_camera(1920, 1080, 1000.0, alt)
            want, _, _ = oracle.filter(tree, cam, 3.0)
            got = s.filter(cam, L.FilterConfig(3.0)).selected
            assert np.array_equal(got, want), alt


def test_filter_mid_trees_leaf_suffix(L, oracle, gpu):
    """Trees large enough that the all-leaf suffix (the fused leaf pass F3)
    starts inside the arena with a ragged last tile, random orbit cameras and
    tau_r: selected lists bit-exact."""
    rng = oracle.rng(77)
    for rep, (nx, depth, k) in enumerate(((6, 3, 8), (9, 3, 8), (5, 4, 6), (13, 3, 8),
                                          (7, 2, 8), (4, 5, 4))):
        tree = L.make_tree(500 + rep, depth, k, 0.5, nx, nx)
        with L.GpuScene(tree) as s:
            for _ in range(6):
                cam = oracle.orbit_camera(rng, 640, 480, oracle.uniform(rng, 3.0, 120.0))
                tau_r = oracle.uniform(rng, 0.5, 40.0)
                want, _, _ = oracle.filter(tree, cam, tau_r)
                got = s.filter(cam, L.FilterConfig(tau_r)).selected
                assert np.array_equal(got, want), (rep, tree.node_count(), tau_r)


def test_filter_serial_random_scenes(L, oracle, gpu):
    """test_filter.cpp:110-140 restated for the device filter_serial: 40 random
    scenes, selection and passes/barriers equal to the oracle's serial filter,
    selection equal to the parallel filter, ascending order."""
    rng = oracle.rng(4242)
    for i in range(40):
        depth = 1 + int(oracle.next_below(rng, 4))
        children = 1 + int(oracle.next_below(rng, 8))
        gamma = float(np.float32(oracle.uniform(rng, 0.3, 0.7)))
        tree = L.make_tree(1000 + i, depth, children, gamma)
        cam = oracle.orbit_camera(rng, 160, 120, oracle.uniform(rng, 3.0, 80.0))
        tau_r = oracle.uniform(rng, 0.5, 60.0)
        oracle.next_below(rng, 4)  # worker count draw
        want, ps, bs = oracle.filter(tree, cam, tau_r, mode=1)
        with L.GpuScene(tree) as s:
            got = s.filter_serial(cam, L.FilterConfig(tau_r))
            par = s.filter(cam, L.FilterConfig(tau_r))
        assert np.array_equal(got.selected, want), i
        assert (got.passes, got.barriers) == (ps, bs), i
        assert np.array_equal(got.selected, par.selected), i
        assert np.all(np.diff(got.selected.astype(np.int64)) > 0)


def test_filter_serial_barriers_per_level(L, oracle, gpu):
    """test_filter.cpp:168-186: the serial filter pays one barrier per
    descended level; everything visible and nothing qualifying selects exactly
    the leaves.  Per-level device times are reported for every level."""
    for depth in (2, 4, 6):
        t = L.make_tree(7, depth, 2, 0.5, 2, 2)
        cam = oracle.front_camera(200, 200)
        cam.translation = (0, 0, 30)
        with L.GpuScene(t) as s:
            lm = np.full(len(t.level_offsets), -1.0)
            rs = s.filter_serial(cam, L.FilterConfig(1e-3), level_ms=lm)
            rp = s.filter(cam, L.FilterConfig(1e-3))
        assert rs.barriers == depth + 1 and rs.passes == depth + 1
        assert np.array_equal(rs.selected, rp.selected)
        assert rs.selected.size == t.node_count() - int(t.level_offsets[depth])
        assert (lm >= 0).all()


def test_filter_serial_descends_only_under_visible_parents(L, oracle, gpu):
    """A child sphere outside its parent's: the serial filter never reaches it
    (its parent is culled) while the parallel filter selects it -- the device
    serial filter keeps the reference's traversal semantics, not the parallel
    rule."""
    t = _hand_tree(L, 1, 8)
    t.mean_x[8] = np.float32(40.0)  # child 8 far to the side of its parent
    t.mean_z[0] = np.float32(-50.0)  # parent behind the camera
    cam = oracle.front_camera(200, 200)
    cam.translation = (-40.0, 0.0, 30.0)
    want_s, ps, _ = oracle.filter(t, cam, 3.0, mode=1)
    want_p, _, _ = oracle.filter(t, cam, 3.0, mode=2)
    with L.GpuScene(t) as s:
        got_s = s.filter_serial(cam, L.FilterConfig(3.0))
        got_p = s.filter(cam, L.FilterConfig(3.0))
    assert np.array_equal(got_s.selected, want_s) and got_s.passes == ps
    assert np.array_equal(got_p.selected, want_p)
    assert not np.array_equal(want_s, want_p)


def test_filter_serial_10m_tree(L, oracle, gpu):
    """cfg 3 tree: serial == parallel == oracle at two altitudes, 4 passes."""
    tree = L.build_synthetic_tree(nx=131, ny=131, seed=1, depth=3, build_seed=7)
    with L.GpuScene(tree) as s:
        for alt in (200.0, 140.0):
            cam = topdown_camera(1920, 1080, 1000.0, alt)
            want, ps, _ = oracle.filter(tree, cam, 3.0, mode=1)
            got = s.filter_serial(cam, L.FilterConfig(3.0))
            assert np.array_equal(got.selected, want) and got.passes == ps == 4
            assert np.array_equal(got.selected, s.filter(cam, L.FilterConfig(3.0)).selected)


def test_filter_frustum_boundary_sweep(L, oracle, gpu):
    """Leaf and internal frustum pre-tests at the planes: the camera slides in
    1e-4 steps so that node spheres cross the side planes inside the FP32
    undecided band (where the FP64 decision must take over); selected lists
    bit-exact at every step."""
    tree = L.make_tree(31, 3, 8, 0.5, 9, 9)  # leaf suffix starts inside the arena
    assert tree.node_count() > 4096
    base = topdown_camera(640, 480, 400.0, 10.0)
    with L.GpuScene(tree) as s:
        for step in range(80):
            cam = topdown_camera(640, 480, 400.0, 10.0)
            tx, ty, tz = base.translation
            cam.translation = (tx + 1e-4 * step, ty - 0.7e-4 * step, tz)
            for tau_r in (3.0, 40.0):
                want, _, _ = oracle.filter(tree, cam, tau_r)
                got = s.filter(cam, L.FilterConfig(tau_r)).selected
                assert np.array_equal(got, want), (step, tau_r)


def test_filter_qpass_threshold_stress(L, oracle, gpu):
    """The FP32-certified qpass pre-test must defer to FP64 whenever a radius
    sits at tau_r: tau_r is set to the exact FP64 radius of visible internal
    nodes and to its neighbouring doubles, selected lists bit-exact."""
    tree = L.build_synthetic_tree(nx=41, ny=42, seed=1, depth=3, build_seed=7)
    n = tree.node_count()
    n_int = int(tree.level_offsets[-1])
    rng = np.random.default_rng(5)
    with L.GpuScene(tree) as s:
        for alt in (50.0, 120.0):
            cam = topdown_camera(1920, 1080, 1000.0, alt)
            vis, _, rad = oracle.mark(tree, cam, 1e300)
            cand = np.flatnonzero(vis[:n_int].astype(bool) & np.isfinite(rad[:n_int]))
            picks = rng.choice(cand, size=min(12, cand.size), replace=False)
            for i in picks:
                r = float(rad[i])
                for tau_r in (r, math.nextafter(r, 0.0), math.nextafter(r, math.inf)):
                    want, _, _ = oracle.filter(tree, cam, tau_r)
                    got = s.filter(cam, L.FilterConfig(tau_r)).selected
                    assert np.array_equal(got, want), (alt, int(i), tau_r)
    assert n > n_int


# ------------------------------------------------------------ preprocess --
def test_prepare_bit_exact(L, oracle, gpu):
    """prepare_gaussians (rasterizer.cpp:48-73): every BlendList field
    bit-identical, all three shrink modes (test_raster.cpp:303-319 fixture)."""
    rng = oracle.rng(40)
    for rep in range(6):
        tree = L.make_tree(5 + rep, 2 + rep % 2, 8, 0.5)
        cam = oracle.orbit_camera(rng, 160, 120, 12.0)
        sel, _, _ = oracle.filter(tree, cam, 6.0)
        with L.GpuScene(tree) as s:
            for mode in (L.ShrinkMode.three_sigma(), L.ShrinkMode.fixed(), L.ShrinkMode.adaptive(0.3)):
                want = oracle.prepare(tree, cam, sel, mode)
                got = s.prepare(cam, sel, mode)
                assert got.size() == want.size()
                for f in L._LIST_F64 + ("depth", "node"):
                    assert getattr(got, f).tobytes() == getattr(want, f).tobytes(), (rep, mode, f)


def test_prepare_near_plane_drop(L, oracle, gpu):
    """test_raster.cpp:280-301: a selected leaf short of the near plane is dropped."""
    t = L.LoDTree.empty(2, 1)
    for i, z in enumerate((10.0, 0.005)):
        t.mean_z[i] = z
        t.scale_x[i] = t.scale_y[i] = t.scale_z[i] = 1.0
        t.quat_w[i] = 1.0
        t.opacity[i] = 0.8
        t.color_r[i] = 1.0
        t.parent[i] = L.ROOT_PARENT
        t.leaf[i] = 1
    cam = oracle.front_camera(64, 64)
    with L.GpuScene(t) as s:
        bl = s.prepare(cam, np.array([0, 1], np.uint32), L.ShrinkMode.three_sigma())
    assert bl.size() == 1 and bl.node[0] == 0
    assert bl.depth[0] == np.float32(10.0)


# --------------------------------------------------------------- binning --
def test_bin_kat(L, gpu):
    """test_raster.cpp:88-118: 9 pairs at (24,24) r=10 on 64x64; r=0; off-screen; corner."""
    grid = L.TileGrid.make(64, 64)
    d = {}
    push_flat(d, 24, 24, 1.0, 0.5, (1, 1, 1), 10.0, np.float32(3.5), 42)
    pairs = L.bin_to_tiles(to_blendlist(d), grid, 64, 64)
    assert len(pairs) == 9
    k = 0
    for ty in range(3):
        for tx in range(3):
            assert pairs[k]["tile"] == grid.tile_id(tx, ty)
            assert pairs[k]["depth"] == np.float32(3.5)
            assert pairs[k]["gaussian"] == 0
            k += 1
    for mx, r in ((24, 0.0), (-100, 10.0)):
        d = {}
        push_flat(d, mx, mx, 1.0, 0.5, (1, 1, 1), r, np.float32(1.0))
        assert len(L.bin_to_tiles(to_blendlist(d), grid, 64, 64)) == 0
    d = {}
    push_flat(d, 63, 63, 1.0, 0.5, (1, 1, 1), 5.0, np.float32(1.0))
    cp = L.bin_to_tiles(to_blendlist(d), grid, 64, 64)
    assert len(cp) == 1 and cp[0]["tile"] == grid.tile_id(3, 3)


def test_bin_random_lists(L, oracle, gpu):
    rng = oracle.rng(2718)
    for rep in range(30):
        w, h, bl = random_micro_scene(oracle, rng)
        want = oracle.bin_to_tiles(bl, w, h)
        got = L.bin_to_tiles(bl, L.TileGrid.make(w, h), w, h)
        assert got.tobytes() == want.tobytes(), rep


# ------------------------------------------------------------------ sort --
def test_sort_100k_kat(L, oracle, gpu):
    """test_raster.cpp:120-135: 100K pairs, 1000 tiles, 50 integer depths
    (plenty of exact ties) equal a stable comparison sort."""
    rng = oracle.rng(99)
    n = 100000
    pairs = np.empty(n, L.PAIR_DTYPE)
    for i in range(n):
        pairs[i] = (oracle.next_below(rng, 1000), np.float32(oracle.next_below(rng, 50)), i)
    expect = pairs[np.lexsort((pairs["depth"], pairs["tile"]))]  # lexsort is stable
    want = pairs.copy()
    oracle.sort_pairs(want)
    assert want.tobytes() == expect.tobytes()
    got = pairs.copy()
    L.sort_pairs(got)
    assert got.tobytes() == expect.tobytes()


def test_sort_hand_cases(L, gpu):
    """test_raster.cpp:137-156."""
    p = np.array([(1, 2.0, 3), (0, 5.0, 1), (1, 2.0, 0), (0, 5.0, 0)], L.PAIR_DTYPE)
    L.sort_pairs(p)
    assert p.tolist() == [(0, 5.0, 1), (0, 5.0, 0), (1, 2.0, 3), (1, 2.0, 0)]
    e = np.empty(0, L.PAIR_DTYPE)
    L.sort_pairs(e)
    one = np.array([(7, 1.0, 0)], L.PAIR_DTYPE)
    L.sort_pairs(one)
    assert one.tolist() == [(7, 1.0, 0)]
    z = np.array([(0, 3.0, 0), (0, 0.0, 1)], L.PAIR_DTYPE)
    L.sort_pairs(z)
    assert z[0]["gaussian"] == 1


def test_sort_big_buckets(L, oracle, gpu):
    """Every bucket-size regime of the per-tile sort against the reference's
    stable LSD sort: register networks (<= 64), the per-tile LSD radix (65..1024:
    1, 2 or 4 keys per thread, 0..4 digit passes), two runs + rank merge in the
    small kernel (<= 2048), 3..16 runs in the big-bucket kernel (<= 16384),
    the global in-place network beyond; one depth only (no digit pass), narrow
    depth bands (with and without ties), wide ones, both mixed in one bucket."""
    rng = np.random.default_rng(5)
    sizes = (33, 64, 65, 100, 255, 256, 257, 400, 511, 512, 513, 777, 1023, 1024, 1025, 1500,
             2047, 2048, 2049, 3000, 4096, 4097, 8263, 16384, 16385, 30000)
    for k, n in enumerate(sizes):
        for depth in ("ties32", "narrow", "ties64", "wide", "one"):
            pairs = np.empty(n, L.PAIR_DTYPE)
            pairs["tile"] = rng.integers(0, 2, n) * 5 if k % 3 == 0 else 3
            if depth == "one":  # every key at one depth: slot order decides alone
                pairs["depth"] = np.float32(7.25)
            elif depth == "ties32":  # 4 distinct depths 2^17 ulps apart
                pairs["depth"] = (100 + rng.integers(0, 4, n)).astype(np.float32)
            elif depth == "ties64":
                pairs["depth"] = rng.integers(0, 300, n).astype(np.float32)
            elif depth == "narrow":
                pairs["depth"] = (50.0 + rng.random(n)).astype(np.float32)
            else:
                pairs["depth"] = (rng.random(n) * 1e4).astype(np.float32)
                pairs["depth"][: n // 7] = np.float32(1e-3)
            pairs["gaussian"] = rng.permutation(n)
            want = pairs.copy()
            oracle.sort_pairs(want)
            got = pairs.copy()
            L.sort_pairs(got)
            assert got.tobytes() == want.tobytes(), (n, depth)


# ----------------------------------------------------------------- blend --
def _blend_pair(L, oracle, d, w, h, exact):
    bl = to_blendlist(d)
    pairs = oracle.bin_to_tiles(bl, w, h)
    oracle.sort_pairs(pairs)
    want = oracle.alpha_blend(pairs, bl, w, h)
    got = L.alpha_blend(pairs, bl, L.TileGrid.make(w, h), w, h, exact=exact).rgb
    return got, want


def test_blend_kats(L, oracle, gpu):
    """test_raster.cpp:158-233 hand cases, exact and fast paths."""
    for exact in (True, False):
        d = {}
        push_flat(d, 8, 8, 0.0, 1.0, (1.0, 0.5, 0.25), 20.0, np.float32(1))
        got, want = _blend_pair(L, oracle, d, 16, 16, exact)
        assert (got[..., 0] == np.float32(0.99)).all()
        assert (got[..., 1] == np.float32(0.5 * 0.99)).all()
        assert (got[..., 2] == np.float32(0.25 * 0.99)).all()
        d = {}
        push_flat(d, 8, 8, 0.0, 0.5, (1, 0, 0), 20.0, np.float32(1), 0)
        push_flat(d, 8, 8, 0.0, 0.5, (0, 1, 0), 20.0, np.float32(2), 1)
        got, want = _blend_pair(L, oracle, d, 16, 16, exact)
        assert (got[..., 0] == 0.5).all() and (got[..., 1] == 0.25).all() and (got[..., 2] == 0).all()
        d = {}
        push_flat(d, 8, 8, 0.0, 0.003, (1, 1, 1), 20.0, np.float32(1), 0)
        push_flat(d, 8, 8, 0.0, 0.5, (1, 0, 0), 20.0, np.float32(2), 1)
        got, want = _blend_pair(L, oracle, d, 16, 16, exact)
        assert got[9, 4, 0] == 0.5
        img = L.alpha_blend(np.empty(0, L.PAIR_DTYPE), to_blendlist({k: [] for k in d}),
                            L.TileGrid.make(33, 17), 33, 17, exact=exact).rgb
        assert (img == 0).all()


def test_blend_termination(L, oracle, gpu):
    d = {}
    for i in range(4):
        push_flat(d, 8, 8, 0.0, 0.99, (1, 1, 1), 20.0, np.float32(i + 1), i)
    got, want = _blend_pair(L, oracle, d, 16, 16, True)
    assert got.tobytes() == want.tobytes()


def test_blend_micro_scenes(L, oracle, gpu):
    """acceptance.cpp:255-288 (#5) micro-scenes: exact path bit-identical,
    fast path within the north-star tolerance."""
    rng = oracle.rng(55)
    for rep in range(50):
        w, h, bl = random_micro_scene(oracle, rng)
        pairs = oracle.bin_to_tiles(bl, w, h)
        oracle.sort_pairs(pairs)
        want = oracle.alpha_blend(pairs, bl, w, h)
        grid = L.TileGrid.make(w, h)
        ex = L.alpha_blend(pairs, bl, grid, w, h, exact=True).rgb
        assert ex.tobytes() == want.tobytes(), rep
        fa = L.alpha_blend(pairs, bl, grid, w, h, exact=False).rgb
        assert max_abs(fa, want) <= IMG_TOL, rep
        # the TMA-staged kernels (same certified per-sample code; k_blend_tma rounds the
        # mean tile-relative instead of block-relative, so its last bits may differ)
        for k in ("tma", "gather4", "wsp"):
            fk = L.alpha_blend(pairs, bl, grid, w, h, blend_kernel=k).rgb
            assert max_abs(fk, want) <= IMG_TOL, (rep, k)
            if k == "wsp":  # same block-relative means and sample order as k_blend_cpa
                assert fk.tobytes() == fa.tobytes(), (rep, k)


def test_blend_needle_splats(L, oracle, gpu):
    """Needle-like splats (2D covariance eigenvalue ratios 1e2..3e4 at any
    angle; the terms of the exponent cancel almost completely): the fast
    path's skip test stays certified -- within the north-star tolerance of the
    oracle -- and the exact path stays bit-identical."""
    rng = np.random.default_rng(77)
    for rep in range(24):
        w, h = 48 + 8 * (rep % 5), 40 + 4 * (rep % 7)
        d: dict = {}
        for i in range(40):
            l1 = 10 ** rng.uniform(2.0, 4.0)
            l2 = rng.uniform(0.3, 1.0)
            th = rng.uniform(0, np.pi)
            c_, s_ = np.cos(th), np.sin(th)
            cov = np.array([[c_ * c_ * l1 + s_ * s_ * l2, c_ * s_ * (l1 - l2)],
                            [c_ * s_ * (l1 - l2), s_ * s_ * l1 + c_ * c_ * l2]])
            con = np.linalg.inv(cov)
            d.setdefault("mean_x", []).append(rng.uniform(0, w))
            d.setdefault("mean_y", []).append(rng.uniform(0, h))
            d.setdefault("conic_a", []).append(con[0, 0])
            d.setdefault("conic_b", []).append(con[0, 1])
            d.setdefault("conic_c", []).append(con[1, 1])
            d.setdefault("opacity", []).append(rng.uniform(0.01, 0.99))
            for c in ("col_r", "col_g", "col_b"):
                d.setdefault(c, []).append(rng.uniform(0, 1))
            d.setdefault("radius", []).append(3.0 * np.sqrt(l1))
            d.setdefault("depth", []).append(np.float32(1.0 + i))
            d.setdefault("node", []).append(i)
        bl = to_blendlist(d)
        pairs = oracle.bin_to_tiles(bl, w, h)
        oracle.sort_pairs(pairs)
        want = oracle.alpha_blend(pairs, bl, w, h)
        grid = L.TileGrid.make(w, h)
        ex = L.alpha_blend(pairs, bl, grid, w, h, exact=True).rgb
        assert ex.tobytes() == want.tobytes(), rep
        fa = L.alpha_blend(pairs, bl, grid, w, h, exact=False).rgb
        assert max_abs(fa, want) <= IMG_TOL, (rep, max_abs(fa, want))
        for k in ("tma", "gather4", "wsp"):
            fk = L.alpha_blend(pairs, bl, grid, w, h, blend_kernel=k).rgb
            assert max_abs(fk, want) <= IMG_TOL, (rep, k, max_abs(fk, want))
            if k == "wsp":
                assert fk.tobytes() == fa.tobytes(), (rep, k)


# ---------------------------------------------------------------- render --
def _check_render(L, oracle, scene, tree, cam, tau_r, mode):
    want = oracle.render(tree, cam, tau_r, mode)
    out = scene.render(cam, L.FilterConfig(tau_r), mode, L.RenderOptions(collect_kpc=True))
    assert out.stats.n_selected == want["n_selected"]
    assert np.array_equal(scene.read_selected(), want["selected"])
    assert out.stats.n_gaussians == want["n_gaussians"]
    assert out.stats.n_pairs == want["n_pairs"]
    assert out.pairs.tobytes() == want["pairs"].tobytes()
    for f in L._LIST_F64 + ("depth", "node"):
        assert getattr(out.gaussians, f).tobytes() == getattr(want["gaussians"], f).tobytes(), f
    # per-gaussian tile counts and per-tile n_gs (metrics.cpp:18-35)
    gl = want["gaussians"]
    n_tiles = L.TileGrid.make(cam.width, cam.height).n_tile()
    pg, pt = scene.read_counts(gl.size(), n_tiles)
    want_pg = np.bincount(want["pairs"]["gaussian"], minlength=gl.size())[: gl.size()]
    want_pt = np.bincount(want["pairs"]["tile"], minlength=n_tiles)[:n_tiles]
    assert np.array_equal(pg, want_pg) and np.array_equal(pt, want_pt)
    # collect_kpc renders through the exact FP64 blend: bit-identical image
    assert out.image.rgb.tobytes() == want["image"].tobytes()
    ex = scene.render(cam, L.FilterConfig(tau_r), mode, L.RenderOptions(exact_blend=True))
    assert ex.image.rgb.tobytes() == want["image"].tobytes()
    # the production frame (flags 0: k_blend_cpa, FP32 + certified FP64 re-check)
    fast = scene.render(cam, L.FilterConfig(tau_r), mode)
    assert fast.stats.n_pairs == want["n_pairs"]
    assert scene.read_pairs().tobytes() == want["pairs"].tobytes()
    err = max_abs(fast.image.rgb, want["image"])
    psnr = oracle.psnr(fast.image.rgb, want["image"]) if err > 0 else math.inf
    assert err <= IMG_TOL, err
    assert psnr > PSNR_MIN, psnr
    return out, want


def test_render_small_scenes(L, oracle, gpu):
    rng = oracle.rng(8)
    tree = L.make_tree(21, 3, 8, 0.5, 3, 3, 2)
    with L.GpuScene(tree) as s:
        for i in range(4):
            cam = oracle.orbit_camera(rng, 200, 150, 14.0)
            for mode in (L.ShrinkMode.three_sigma(), L.ShrinkMode.fixed(), L.ShrinkMode.adaptive(0.1)):
                _check_render(L, oracle, s, tree, cam, 4.0, mode)


def test_render_cfg1(L, oracle, gpu):
    """cfg 1: 99,937 nodes, 800x600, fx=100, z=12."""
    tree = L.build_synthetic_tree(nx=37, ny=37, seed=1, depth=2, build_seed=7)
    assert tree.node_count() == 99937
    cam = oracle.front_camera(800, 600, 100.0)
    cam.translation = (0, 0, 12)
    with L.GpuScene(tree) as s:
        out, want = _check_render(L, oracle, s, tree, cam, 3.0, L.ShrinkMode.three_sigma())
    assert want["n_selected"] == 86321 and want["n_pairs"] == 303131  # survey probe numbers


def test_render_black_and_errors(L, oracle, gpu):
    """test_raster.cpp:321-330, :390-399."""
    tree = L.make_tree(3, 2, 8, 0.5)
    cam = oracle.front_camera(96, 64)
    cam.translation = (0, 0, -100)
    with L.GpuScene(tree) as s:
        out = s.render(cam, L.FilterConfig(3.0), L.ShrinkMode.three_sigma())
        assert out.stats.n_selected == 0 and out.stats.n_pairs == 0
        assert (out.image.rgb == 0).all()
        for bad in (0.0, 1.0):
            with pytest.raises(L.ValidationError):
                s.render(cam, L.FilterConfig(3.0), L.ShrinkMode.adaptive(bad))


def test_render_deterministic_and_overflow_regrow(L, oracle, gpu):
    """Byte-identical frames on repeat; a deliberately tiny pair buffer is
    grown and the frame re-rendered with identical output."""
    tree = L.make_tree(33, 3, 8, 0.5, 3, 3, 3)
    rng = oracle.rng(5)
    cam = oracle.orbit_camera(rng, 200, 150, 16.0)
    with L.GpuScene(tree) as s:
        a = s.render(cam, L.FilterConfig(5.0), L.ShrinkMode.three_sigma()).image.rgb.copy()
        b = s.render(cam, L.FilterConfig(5.0), L.ShrinkMode.three_sigma()).image.rgb.copy()
        assert a.tobytes() == b.tobytes()
    with L.GpuScene(tree) as s2:
        # the scene starts with max(4N, 1M) pairs: force an overflow path by a huge
        # close-up frame that needs more pairs than nodes * 4
        cam2 = oracle.front_camera(1024, 1024, 2000.0)
        cam2.translation = (0, 0, 9.0)
        want = oracle.render(tree, cam2, 1e9, L.ShrinkMode.three_sigma())
        out = s2.render(cam2, L.FilterConfig(1e9), L.ShrinkMode.three_sigma())
        assert out.stats.n_pairs == want["n_pairs"]
        assert max_abs(out.image.rgb, want["image"]) <= IMG_TOL


def test_render_cfg3_frame(L, oracle, gpu):
    """A full cfg 3 frame (10M nodes, 1080p, altitude 200): everything bit-exact
    against the oracle, image within tolerance."""
    tree = L.build_synthetic_tree(nx=131, ny=131, seed=1, depth=3, build_seed=7)
    cam = topdown_camera(1920, 1080, 1000.0, 200.0)
    with L.GpuScene(tree) as s:
        out, want = _check_render(L, oracle, s, tree, cam, 3.0, L.ShrinkMode.three_sigma())
    assert want["n_pairs"] > 1_000_000


def test_render_batch_matches_single_frames(L, oracle, gpu):
    """lodgs_gpu_render_batch (pipelined, double-buffered) returns the same images and
    stats as one lodgs_gpu_render per frame."""
    import ctypes as C

    tree = L.make_tree(21, 3, 8, 0.5, 3, 3, 2)
    rng = oracle.rng(17)
    cams = [oracle.orbit_camera(rng, 200, 150, 14.0) for _ in range(5)]
    for c in cams:
        c.fx = c.fy = 150.0  # one intrinsics set: batch frames share the image size
    imgs = [np.empty((150, 200, 3), np.float32) for _ in cams]
    with L.GpuScene(tree) as s:
        stats = s.render_batch(cams, L.FilterConfig(4.0), L.ShrinkMode.three_sigma(),
                               host_ptrs=[im.ctypes.data for im in imgs])
        for cam, im, st in zip(cams, imgs, stats):
            one = s.render(cam, L.FilterConfig(4.0), L.ShrinkMode.three_sigma())
            assert im.tobytes() == one.image.rgb.tobytes()
            assert st.n_pairs == one.stats.n_pairs and st.n_selected == one.stats.n_selected
            want = oracle.render(tree, cam, 4.0, L.ShrinkMode.three_sigma())
            assert max_abs(im, want["image"]) <= IMG_TOL


def test_render_async_frames_in_flight(L, oracle, gpu):
    """lodgs_gpu_render_async with 4, 3, 2 and 1 frames in flight (the scene
    and up to three twin contexts): every frame's image and the run totals
    equal the synchronous renders; the last frame is what sync() reports and
    read_image() returns; more than 12 is refused."""
    tree = L.make_tree(23, 3, 8, 0.5, 4, 4, 2)
    rng = oracle.rng(29)
    cams = [oracle.orbit_camera(rng, 200, 150, 16.0) for _ in range(7)]
    for c in cams:
        c.fx = c.fy = 150.0
    mode = L.ShrinkMode.three_sigma()
    with L.GpuScene(tree) as s:
        ref = [s.render(cam, L.FilterConfig(4.0), mode) for cam in cams]
        for inflight in (4, 3, 2, 1, 8, 12, 6, 4):
            s.set_inflight(inflight)
            p = s.params(L.FilterConfig(4.0), mode, L.RenderOptions())
            imgs = [np.empty((150, 200, 3), np.float32) for _ in cams]
            s.take_totals()
            for cam, im in zip(cams, imgs):
                s.render_async(cam, p, im.ctypes.data)
            last = s.sync()
            frames, sel, pairs = s.take_totals()
            assert frames == len(cams)
            assert sel == sum(r.stats.n_selected for r in ref)
            assert pairs == sum(r.stats.n_pairs for r in ref)
            for im, r in zip(imgs, ref):
                assert im.tobytes() == r.image.rgb.tobytes()
            assert last.n_pairs == ref[-1].stats.n_pairs
            assert s.read_image(cams[-1]).tobytes() == ref[-1].image.rgb.tobytes()
        for bad in (0, 13):
            with pytest.raises(L.ValidationError):
                s.set_inflight(bad)


def test_cfg4_50m_4k(L, oracle, gpu):
    """cfg 4 scale (50,142,872 nodes, 3840x2160, fx = 2000): selected list
    bit-exact at altitude 300, and a full frame at altitude 400 (pairs, counts,
    exact image bit-identical, fast image within tolerance)."""
    tree = L.build_synthetic_tree(nx=103, ny=104, seed=1, depth=4, build_seed=7)
    assert tree.node_count() == 50142872
    with L.GpuScene(tree) as s:
        cam = topdown_camera(3840, 2160, 2000.0, 300.0)
        want, _, _ = oracle.filter(tree, cam, 3.0)
        assert np.array_equal(s.filter(cam, L.FilterConfig(3.0)).selected, want)
        cam = topdown_camera(3840, 2160, 2000.0, 400.0)
        _check_render(L, oracle, s, tree, cam, 3.0, L.ShrinkMode.three_sigma())


# ------------------------------------------------------- kpc / calibration --
def test_kpc_bit_identical(L, oracle, gpu):
    """collect_kpc (rasterizer.hpp:86-96): per-pair kpc in the reference's 4-lane
    order (blend_scalar.cpp:16-54), bit-identical; image exact; ragged edge tiles."""
    rng = oracle.rng(66)
    tree = L.make_tree(13, 2, 8, 0.5, 3, 3, 2)
    with L.GpuScene(tree) as s:
        for w, h in ((160, 120), (150, 100), (33, 17)):
            cam = oracle.orbit_camera(rng, w, h, 12.0)
            for mode in (L.ShrinkMode.three_sigma(), L.ShrinkMode.adaptive(0.2)):
                want = oracle.render(tree, cam, 6.0, mode, collect_kpc=True)
                out = s.render(cam, L.FilterConfig(6.0), mode, L.RenderOptions(collect_kpc=True))
                assert out.pairs.tobytes() == want["pairs"].tobytes()
                kw = want["kpc"] if want["kpc"] is not None else np.empty(0)
                assert out.kpc.tobytes() == kw.tobytes()
                assert out.image.rgb.tobytes() == want["image"].tobytes()


def _oracle_calibrate(oracle, tree, views, lambda_g, tau_r, L):
    per = []
    for v in views:
        r = oracle.render(tree, v, tau_r, L.ShrinkMode.three_sigma(), collect_kpc=True)
        if r["n_pairs"]:
            per.append(oracle.view_gtc(r["pairs"], r["kpc"]))
    mean = 0.0
    for g in per:
        mean += g
    mean /= len(per)
    return per, mean, lambda_g / mean


def test_shrink_study_acceptance_7_8_9(L, oracle, gpu):
    """acceptance.cpp:343-433 (#7-#9) on the GPU: calibrate (tau bit-exact against
    the oracle restatement of metrics.cpp:94-108), then 3-sigma / fixed / adaptive
    renders of 5 orbit views with tau_R = 16 (pair counts, kpc, images exact)."""
    tree = L.make_tree(8008, 2, 8, 0.5, 4, 4, 4)
    rng = oracle.rng(88)
    views = [oracle.orbit_camera(rng, 160, 120, 12.0) for _ in range(5)]
    per, mean, tau = _oracle_calibrate(oracle, tree, views, 0.2, 16.0, L)
    with L.GpuScene(tree) as s:
        rep = s.calibrate(views, 0.2, L.FilterConfig(16.0))
        assert rep.n_views == len(per)
        assert rep.per_view.tolist() == per
        assert rep.scene_mean == mean and rep.tau == tau
        totals = {"3s": 0, "fixed": 0, "adaptive": 0}
        low = {"3s": 0, "adaptive": 0}
        worst = float("inf")
        for v in views:
            imgs = {}
            for name, mode in (("3s", L.ShrinkMode.three_sigma()), ("fixed", L.ShrinkMode.fixed()),
                               ("adaptive", L.ShrinkMode.adaptive(tau))):
                want = oracle.render(tree, v, 16.0, mode, collect_kpc=True)
                out = s.render(v, L.FilterConfig(16.0), mode, L.RenderOptions(collect_kpc=True))
                assert out.stats.n_pairs == want["n_pairs"]
                kw = want["kpc"] if want["kpc"] is not None else np.empty(0)
                assert out.kpc.tobytes() == kw.tobytes()
                totals[name] += out.stats.n_pairs
                if name in low:
                    low[name] += int((out.kpc < 0.05).sum())
                imgs[name] = out.image.rgb
            worst = min(worst, oracle.psnr(imgs["adaptive"], imgs["3s"]))
    # reference gate outputs on this fixture (acceptance #8/#9)
    assert (totals["3s"], totals["fixed"], totals["adaptive"]) == (9921, 9916, 6038)
    assert (low["3s"], low["adaptive"]) == (5065, 1680)
    assert round(tau, 4) == 0.1050 and round(worst, 1) == 49.1
