"""CPU tests (no GPU): the oracle pinned against the reference, the host logic,
and the C ABI surface.

* Golden fixtures (tests/golden/golden_v1.npz, generated from the reference
  library by tests/golden/make_golden.py) pin the oracle wherever the
  reference itself is absent.
* Where oracle/_ref exists (this container), the oracle is also compared
  live against the reference on the reference's own test configurations.
"""
import ctypes as C
import hashlib
import math
import os
import re

import numpy as np
import pytest

from helpers import ACCEPT_SHAPES, acceptance_filter_configs, push_flat, random_micro_scene, to_blendlist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = np.load(os.path.join(ROOT, "tests", "golden", "golden_v1.npz"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------- golden fixtures --
def test_golden_exp_mx(oracle):
    """fastexp.hpp:38-50: identical to the reference bit for bit."""
    ys = np.array([oracle.exp_mx(float(x)) for x in GOLDEN["exp_x"]])
    assert ys.tobytes() == GOLDEN["exp_y"].tobytes()
    # test_kernels.cpp:82-101
    assert oracle.exp_mx(0.0) == 1.0
    assert oracle.exp_mx(-45.0) == oracle.exp_mx(-30.0)
    assert oracle.exp_mx(-30.0) < 1.0 / 255.0
    xs = np.random.default_rng(606).uniform(-30, 0, 20000)
    worst = max(abs(oracle.exp_mx(x) - math.exp(x)) / math.exp(x) for x in xs)
    assert worst < 1e-15


def test_golden_effective_radius(oracle):
    for sigma, op, kind, tau, want in GOLDEN["eff_radius"]:
        got = oracle.effective_radius(sigma, np.float32(op), int(kind), tau)
        assert got == want


def test_effective_radius_closed_forms(oracle):
    """test_raster.cpp:40-86 / acceptance.cpp:202-233 (#4)."""
    assert oracle.effective_radius(1.0, np.float32(0.7), 0, 0.0) == 3.0
    assert oracle.effective_radius(1.0, np.float32(0.25), 2, 0.25) == 0.0
    assert oracle.effective_radius(1.0, np.float32(1.0), 1, 1 / 255) == 3.0
    got = oracle.effective_radius(2.0, np.float32(0.5), 2, 0.2)
    assert got == pytest.approx(2.0 * math.sqrt(2.0 * math.log(2.5)), rel=1e-12)
    with pytest.raises(Exception):
        oracle.effective_radius(1.0, np.float32(0.5), 2, 0.0)
    rng = oracle.rng(44)
    for _ in range(1000):
        tau = oracle.uniform(rng, 0.01, 0.9)
        cap = min(math.exp(4.5) - 0.1, 1.0 / tau)
        a0 = tau * oracle.uniform(rng, 1.001, cap)
        sigma = oracle.uniform(rng, 0.3, 8.0)
        r = oracle.effective_radius(sigma, np.float32(a0), 2, tau)
        edge = float(np.float32(a0)) * math.exp(-r * r / (2 * sigma * sigma))
        assert abs(edge - tau) <= 1e-6


def test_golden_scenes(L, oracle):
    """Whole-frame outputs of the reference (selected, sorted pairs, image,
    kpc, BlendList) reproduced bit for bit by the oracle."""
    from golden.make_golden import SCENES

    for i, (seed, depth, k, gamma, nx, ny, cong, cseed, w, h, dist, tau_r, kind, tau) in enumerate(SCENES):
        tree = L.make_tree(seed, depth, k, gamma, nx, ny, cong)
        cam = oracle.orbit_camera(oracle.rng(cseed), w, h, dist)
        r = oracle.render(tree, cam, tau_r, L.ShrinkMode(kind, tau), collect_kpc=True)
        counts = GOLDEN[f"scene{i}_counts"]
        assert (r["n_selected"], r["n_pairs"], r["n_gaussians"]) == tuple(counts)
        hs = GOLDEN[f"scene{i}_hashes"]
        lh = hashlib.sha256(b"".join(np.ascontiguousarray(getattr(r["gaussians"], f)).tobytes()
                                     for f in L._LIST_F64 + ("depth", "node"))).hexdigest()
        kpc = r["kpc"] if r["kpc"] is not None else np.empty(0)
        assert [sha(r["selected"]), sha(r["pairs"]), sha(r["image"]), sha(kpc), lh] == list(hs), i


def test_golden_sort_kat(L, oracle):
    """test_raster.cpp:120-135: 100K pairs equal a stable comparison sort."""
    rng = oracle.rng(99)
    n = 100000
    pairs = np.empty(n, L.PAIR_DTYPE)
    for i in range(n):
        pairs[i] = (oracle.next_below(rng, 1000), np.float32(oracle.next_below(rng, 50)), i)
    assert sha(pairs) == GOLDEN["sort_in_hash"][0]
    expect = pairs[np.lexsort((pairs["depth"], pairs["tile"]))]
    oracle.sort_pairs(pairs)
    assert pairs.tobytes() == expect.tobytes()
    assert sha(pairs) == GOLDEN["sort_out_hash"][0]


def test_sort_hand_cases(L, oracle):
    """test_raster.cpp:137-156."""
    p = np.array([(1, 2.0, 3), (0, 5.0, 1), (1, 2.0, 0), (0, 5.0, 0)], L.PAIR_DTYPE)
    oracle.sort_pairs(p)
    assert p.tolist() == [(0, 5.0, 1), (0, 5.0, 0), (1, 2.0, 3), (1, 2.0, 0)]
    z = np.array([(0, 3.0, 0), (0, 0.0, 1)], L.PAIR_DTYPE)
    oracle.sort_pairs(z)
    assert z[0]["gaussian"] == 1


def test_golden_micro_blends(oracle):
    rng = oracle.rng(55)
    for rep in range(50):
        w, h, bl = random_micro_scene(oracle, rng)
        p = oracle.bin_to_tiles(bl, w, h)
        oracle.sort_pairs(p)
        assert sha(oracle.alpha_blend(p, bl, w, h)) == GOLDEN["micro_hashes"][rep], rep


def test_blend_kats(oracle):
    """test_raster.cpp:158-233 on the oracle."""
    def run(d, w=16, h=16):
        bl = to_blendlist(d)
        p = oracle.bin_to_tiles(bl, w, h)
        oracle.sort_pairs(p)
        return oracle.alpha_blend(p, bl, w, h, kpc=True)

    d = {}
    push_flat(d, 8, 8, 0.0, 1.0, (1.0, 0.5, 0.25), 20.0, np.float32(1))
    img, kpc = run(d)
    assert (img[..., 0] == np.float32(0.99)).all() and kpc[0] == pytest.approx(256 * 0.99)
    d = {}
    push_flat(d, 8, 8, 0.0, 0.5, (1, 0, 0), 20.0, np.float32(1), 0)
    push_flat(d, 8, 8, 0.0, 0.5, (0, 1, 0), 20.0, np.float32(2), 1)
    img, kpc = run(d)
    assert (img[..., 0] == 0.5).all() and (img[..., 1] == 0.25).all()
    assert kpc.tolist() == [128.0, 64.0]
    d = {}
    for i in range(4):
        push_flat(d, 8, 8, 0.0, 0.99, (1, 1, 1), 20.0, np.float32(i + 1), i)
    _, kpc = run(d)
    assert kpc[0] > 0 and kpc[1] > 0 and kpc[2] > 0 and kpc[3] == 0 and kpc[2] < kpc[1]


def test_calibration_arithmetic(L, oracle):
    """acceptance.cpp:343-358 (#7): G_v == 6 exactly."""
    pairs = np.array([(0, 1.0, 0), (0, 2.0, 1)], L.PAIR_DTYPE)
    assert oracle.view_gtc(pairs, np.array([10.0, 2.0])) == 6.0


# -------------------------------------------------- oracle vs reference --
def test_filter_three_way_acceptance(L, oracle, ref):
    """acceptance.cpp:93-135 (#1): oracle-parallel == reference oracle ==
    reference serial == reference parallel on the 208 configurations; the
    oracle's serial descent matches the reference's barrier counts."""
    count = 0
    handles = {}
    for tree, cam, tau_r in acceptance_filter_configs(oracle):
        h = handles.get(id(tree))
        if h is None:
            for old in handles.values():
                ref.free_tree(old)
            handles = {id(tree): ref.tree_from(tree)}
            h = handles[id(tree)]
        n = tree.node_count()
        mine, p, b = oracle.filter(tree, cam, tau_r)
        assert (p, b) == (2, 2)
        for mode in (0, 1, 2):
            want, rp, rb = ref.filter(h, n, cam, tau_r, mode=mode)
            assert np.array_equal(mine, want), (count, mode)
        s, sp, sb = oracle.filter(tree, cam, tau_r, mode=1)
        _, rp, rb = ref.filter(h, n, cam, tau_r, mode=1)
        assert (sp, sb) == (rp, rb) and np.array_equal(s, mine)
        count += 1
    for old in handles.values():
        ref.free_tree(old)
    assert count == 208


def test_mark_bit_identical_vs_reference(L, oracle, ref):
    """test_kernels.cpp:128-171: scalar and AVX2 reference marks == oracle marks."""
    rng = oracle.rng(11)
    for rep in range(12):
        tree = L.make_tree(200 + rep, 2 + rep % 3, 8, 0.5, 3, 3)
        h = ref.tree_from(tree)
        n = tree.node_count()
        cam = oracle.orbit_camera(rng, 320, 240, oracle.uniform(rng, 2.0, 60.0))
        tau_r = oracle.uniform(rng, 0.5, 40.0)
        v, q, r = oracle.mark(tree, cam, tau_r)
        for backend in (0, 1):
            v2, q2, r2 = ref.mark(h, n, cam, tau_r, backend=backend)
            assert np.array_equal(v, v2) and np.array_equal(q, q2) and r.tobytes() == r2.tobytes()
        ref.free_tree(h)


def test_stages_bit_identical_vs_reference(L, oracle, ref):
    rng = oracle.rng(40)
    for rep in range(6):
        tree = L.make_tree(5 + rep, 2 + rep % 2, 8, 0.5)
        h = ref.tree_from(tree)
        cam = oracle.orbit_camera(rng, 160, 120, 12.0)
        sel, _, _ = oracle.filter(tree, cam, 6.0)
        for mode in (L.ShrinkMode.three_sigma(), L.ShrinkMode.fixed(), L.ShrinkMode.adaptive(0.3)):
            a = oracle.prepare(tree, cam, sel, mode)
            b = ref.prepare(h, cam, sel, mode)
            for f in L._LIST_F64 + ("depth", "node"):
                assert getattr(a, f).tobytes() == getattr(b, f).tobytes()
            pa, pb = oracle.bin_to_tiles(a, 160, 120), ref.bin_to_tiles(b, 160, 120)
            assert pa.tobytes() == pb.tobytes()
            oracle.sort_pairs(pa)
            ref.sort_pairs(pb)
            assert pa.tobytes() == pb.tobytes()
            ia, ka = oracle.alpha_blend(pa, a, 160, 120, kpc=True)
            ib, kb = ref.alpha_blend(pb, b, 160, 120, workers=3, kpc=True)
            assert ia.tobytes() == ib.tobytes() and ka.tobytes() == kb.tobytes()
        ref.free_tree(h)


def test_render_cfg1_vs_reference(L, oracle, ref):
    """cfg 1: 99,937 nodes, 800x600: identical image, pairs
    and counts; survey probe numbers reproduced."""
    tree = L.build_synthetic_tree(nx=37, ny=37, seed=1, depth=2, build_seed=7)
    h = ref.tree_from(tree)
    cam = oracle.front_camera(800, 600, 100.0)
    cam.translation = (0, 0, 12)
    a = oracle.render(tree, cam, 3.0, L.ShrinkMode.three_sigma(), collect_kpc=True)
    b = ref.render(h, cam, 3.0, L.ShrinkMode.three_sigma(), workers=4, collect_kpc=True)
    ref.free_tree(h)
    assert (a["n_selected"], a["n_pairs"]) == (86321, 303131)
    assert (b["n_selected"], b["n_pairs"]) == (86321, 303131)
    assert a["image"].tobytes() == b["image"].tobytes()
    assert a["pairs"].tobytes() == b["pairs"].tobytes()
    assert a["kpc"].tobytes() == b["kpc"].tobytes()


def test_calibrate_vs_reference(L, oracle, ref):
    """metrics.cpp:94-108: the oracle's calibration (kpc -> tile GTC -> view GTC ->
    tau) equals the reference's calibrate bit for bit (acceptance #8 fixture)."""
    import ctypes as C

    from test_gpu_parity import _oracle_calibrate

    tree = L.make_tree(8008, 2, 8, 0.5, 4, 4, 4)
    rng = oracle.rng(88)
    views = [oracle.orbit_camera(rng, 160, 120, 12.0) for _ in range(5)]
    per, mean, tau = _oracle_calibrate(oracle, tree, views, 0.2, 16.0, L)
    h = ref.tree_from(tree)
    vc = (L.CameraC * 5)(*[v.to_c() for v in views])
    t, sg, nu = C.c_double(), C.c_double(), C.c_uint32()
    pv = np.zeros(5)
    hist = np.zeros(5, np.uint64)
    rc = ref.lib.ref_calibrate(h, vc, 5, 0.2, 16.0, 2, C.byref(t), C.byref(sg),
                               pv.ctypes.data_as(C.POINTER(C.c_double)), C.byref(nu),
                               hist.ctypes.data_as(C.c_void_p))
    ref.free_tree(h)
    assert rc == 0
    assert (t.value, sg.value) == (tau, mean)
    assert pv[: nu.value].tolist() == per
    assert round(tau, 4) == 0.1050


# --------------------------------------------------------- host logic --
def test_generator_matches_reference_golden(L):
    """The product's synthetic scene builder (host_util.cpp) reproduces the
    reference generator (tree_builder.cpp:75-174) bit for bit."""
    from golden.make_golden import TREES

    for i, (nx, ny, seed, cong, depth, gamma, k, bseed) in enumerate(TREES):
        t = L.build_synthetic_tree(nx=nx, ny=ny, seed=seed, congestion=cong, depth=depth,
                                   shrink_factor=gamma, children_per_node=k,
                                   build_seed=bseed & 0xFFFFFFFFFFFFFFFF)
        assert t.node_count() == GOLDEN[f"tree{i}_n"][0]
        blob = np.concatenate([getattr(t, f).view(np.uint8)
                               for f in L._FIELDS + ("parent", "leaf", "level_offsets")])
        assert sha(blob) == GOLDEN[f"tree{i}_hash"][0], i
        assert L.validate_tree(t) == 0


def test_generator_matches_reference_live(L, ref):
    for seed, depth, k, gamma, nx, ny, cong in ((11, 3, 5, 0.41, 2, 3, 2), (3, 4, 2, 0.7, 2, 2, 1)):
        h, rt = ref.make_tree(seed, depth, k, np.float32(gamma), nx, ny, cong)
        t = L.make_tree(seed, depth, k, float(np.float32(gamma)), nx, ny, cong)
        ref.free_tree(h)
        for f in L._FIELDS + ("parent", "leaf", "level_offsets"):
            assert getattr(t, f).tobytes() == getattr(rt, f).tobytes(), f


def test_camera_path_matches_reference_golden(L):
    import bench

    frames = bench.flythrough(L)
    arr = np.array([[*f.rotation, *f.translation, f.fx, f.fy, f.cx, f.cy, f.near, f.far]
                    for f in frames])
    assert len(frames) == 300
    assert arr.tobytes() == GOLDEN["path_frames"].tobytes()


def test_camera_geom_matches_oracle(L, oracle):
    rng = oracle.rng(3)
    for _ in range(20):
        cam = oracle.orbit_camera(rng, 321, 200, oracle.uniform(rng, 3.0, 60.0))
        assert L.camera_geom(cam).tobytes() == oracle.camera_geom(cam).tobytes()


def test_validation_catches_corruptions(L, oracle):
    """acceptance.cpp:519-542 (#11): 60 seeded single-field corruptions."""
    for i in range(60):
        t = L.make_tree(7000 + i, 2, 4, 0.5, 2, 2)
        assert L.validate_tree(t) == 0
        r = oracle.rng(oracle.lib.orc_mix_seed(42, i))
        n = int(oracle.next_below(r, t.node_count()))
        case = i % 8
        if case == 0:
            t.scale_x[n] = -1.0
        elif case == 1:
            t.opacity[n] = 0.0
        elif case == 2:
            t.opacity[n] = 1.5
        elif case == 3:
            t.quat_w[n] = 3.0
        elif case == 4:
            t.color_r[n] = 2.0
        elif case == 5:
            t.mean_y[n] = np.nan
        elif case == 6:
            t.leaf[n] = 0 if t.leaf[n] else 1
        else:
            t.parent[n] = 1 if t.parent[n] == L.ROOT_PARENT else L.ROOT_PARENT
        assert L.validate_tree(t) > 0, i
        with pytest.raises(L.ValidationError):
            L.require_valid(t)


def test_validation_counts_match_reference(L, ref):
    t = L.make_tree(7, 2, 4, 0.5, 2, 2)
    t.opacity[3] = 2.0
    t.scale_y[5] = 0.0
    h = ref.tree_from(t)
    assert ref.validate(h) == L.validate_tree(t) == 2
    ref.free_tree(h)


def test_camera_validation(L):
    lib = L.load_library()
    cam = L.Camera(64, 64, 100, 100, 32, 32).to_c()
    n = C.c_uint64(0)
    assert lib.lodgs_validate_camera(C.byref(cam), C.byref(n), None, 0) == 0 and n.value == 0
    cam.fx = 0.0
    cam.rotation[0] = 2.0
    assert lib.lodgs_validate_camera(C.byref(cam), C.byref(n), None, 0) == 0 and n.value == 2


# ------------------------------------------------------------- the ABI --
def test_abi_exports_every_declared_symbol(L):
    """include/lodgs_gpu.h declares exactly the lodgs_* symbols the .so exports."""
    header = open(os.path.join(ROOT, "include", "lodgs_gpu.h")).read()
    declared = set(re.findall(r"LODGS_API\s+(?:const\s+char\s*\*|int)\s*(lodgs_\w+)\s*\(", header))
    lib = L.load_library()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(L.ABI_SYMBOLS)
    assert lib.lodgs_gpu_abi_version() == 1
    # input generation (synthetic trees, camera paths) is a separate library
    synth_h = open(os.path.join(ROOT, "include", "lodgs_synth.h")).read()
    synth = set(re.findall(r"LODGS_API\s+(?:const\s+char\s*\*|int)\s*(lodgs_\w+)\s*\(", synth_h))
    assert synth == set(L.SYNTH_SYMBOLS)
    slib = L.load_synth_library()
    for name in synth:
        assert hasattr(slib, name) and not hasattr(lib, name), name


def test_no_cpu_fallback_without_device(L):
    """Compute entry points fail loudly (status 4) when no CUDA device is usable."""
    if L.device_count() > 0:
        pytest.skip("a device is present")
    t = L.make_tree(1, 1, 8, 0.5, 1, 1)
    with pytest.raises(L.CudaError):
        L.GpuScene(t)
    pairs = np.array([(1, 2.0, 3), (0, 5.0, 1)], L.PAIR_DTYPE)
    with pytest.raises(L.CudaError):
        L.sort_pairs(pairs)


def test_render_rejects_bad_tau(L):
    t = L.make_tree(1, 1, 8, 0.5, 1, 1)
    cam = L.Camera(64, 64, 100, 100, 32, 32)
    for bad in (0.0, 1.0):
        with pytest.raises(L.ValidationError):
            L.render(t, cam, L.FilterConfig(3.0), L.ShrinkMode.adaptive(bad))


# ------------------------------------------------------- LDGS scene files --
@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_ldgs_tool")),
                    reason="oracle/_ref not built")
def test_ldgs_writer_matches_reference_save_scene(L, tmp_path):
    """tests/helpers.write_ldgs (the restated save_binary) writes the bytes the
    reference's save_scene writes (scene_io.cpp:55-84), and the reference
    loads them back."""
    from helpers import ref_ldgs, write_ldgs

    for nx, ny, seed, depth, bseed in ((5, 5, 1, 3, 7), (3, 4, 9, 2, 1), (2, 2, 3, 4, 5)):
        ref_path = tmp_path / f"ref_{nx}_{depth}.ldgs"
        assert ref_ldgs("save", ref_path, nx, ny, seed, depth, bseed) == "SAVED"
        tree = L.build_synthetic_tree(nx=nx, ny=ny, seed=seed, depth=depth, build_seed=bseed)
        mine = tmp_path / f"mine_{nx}_{depth}.ldgs"
        write_ldgs(tree, mine)
        assert mine.read_bytes() == ref_path.read_bytes()
        ok, n, levels, _ = ref_ldgs("load", mine).split()
        assert ok == "OK" and int(n) == tree.node_count() and int(levels) == len(tree.level_offsets)


def test_integration_shim_compiles_against_reference_headers(tmp_path):
    """INTEGRATION.md's reference-side C++ shim (lodgs::render over the C ABI)
    type-checks against the reference's own headers and include/lodgs_gpu.h."""
    import shutil
    import subprocess

    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc) or not shutil.which("g++"):
        pytest.skip("reference headers or g++ absent")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "INTEGRATION.md")).read()
    start = text.index("```cpp\n// proj/src/rasterizer_b200.cpp") + len("```cpp\n")
    src = os.path.join(root, "integration", "rasterizer_b200.cpp")
    # the listing in INTEGRATION.md is the file that oracle/_ref/shim_check links and runs
    assert text[start:text.index("```", start)] == open(src).read()
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{ref_inc}",
                        f"-I{os.path.join(root, 'include')}", str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
