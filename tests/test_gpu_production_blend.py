"""The production frame path -- k_blend_cpa, the kernel bench.py times -- against the
reference renderer itself (oracle/_ref, compiled from /root/reference's sources) on
the BASELINE.json configurations.

Every frame here renders WITHOUT collect_kpc / exact_blend (flags 0), through the
entry points the bench and the drop-in shim use: lodgs_gpu_render_async with four
frames in flight, lodgs_gpu_render_batch (pipelined, image ring) and the synchronous
lodgs_gpu_render.  Per frame: n_selected and n_pairs equal, image max-abs <= 1e-3 per
channel and PSNR > 60 dB against the reference image (north_star); on the synchronous
renders the sorted (tile, depth, gaussian) sequence is compared bit for bit as well.

Reference: lodgs::render (rasterizer.cpp:167-213); the blend it is compared with is
alpha_blend -> blend_scalar (rasterizer.cpp:137-165, blend_scalar.cpp:13-55).
"""
import os
import sys

import numpy as np
import pytest

from helpers import max_abs, topdown_camera

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-3   # BASELINE.json north_star: max-abs 1e-3 per channel
PSNR_MIN = 60.0  # ... and PSNR > 60 dB
THREADS = os.cpu_count() or 1
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    sys.path.insert(0, ROOT)
    import bench

    return bench


def _compare(ref, rh, cam, tau_r, mode, img, st, what, want=None):
    if want is None:
        want = ref.render(rh, cam, tau_r, mode, workers=THREADS)
    if st is not None:
        assert st.n_selected == want["n_selected"], what
        assert st.n_pairs == want["n_pairs"], what
    err = max_abs(img, want["image"])
    psnr = ref.psnr(img, want["image"]) if err > 0 else float("inf")
    assert err <= IMG_TOL, (what, err)
    assert psnr > PSNR_MIN, (what, psnr)
    return want, err, psnr


def _async_frames(L, scene, cams, tau_r, mode, blend_kernel="cpa"):
    """Four frames in flight (render_async), every image to its own host buffer."""
    scene.set_inflight(4)
    p = scene.params(L.FilterConfig(tau_r), mode, L.RenderOptions(blend_kernel=blend_kernel))
    imgs = [np.empty((c.height, c.width, 3), np.float32) for c in cams]
    for cam, im in zip(cams, imgs):
        scene.render_async(cam, p, im.ctypes.data)
    scene.sync()
    return imgs


def _views(L, scene, cams, tau_r, mode):
    imgs = [np.empty((c.height, c.width, 3), np.float32) for c in cams]
    p = scene.params(L.FilterConfig(tau_r), mode, L.RenderOptions())
    scene.render_views_async(cams, p, host_ptrs=[im.ctypes.data for im in imgs])
    scene.sync()
    return imgs


def _batch_frames(L, scene, cams, tau_r, mode):
    imgs = [np.empty((c.height, c.width, 3), np.float32) for c in cams]
    stats = scene.render_batch(cams, L.FilterConfig(tau_r), mode,
                               host_ptrs=[im.ctypes.data for im in imgs])
    return imgs, stats


def _sync_check(L, ref, rh, scene, cam, tau_r, mode, what):
    """One synchronous production render: image within tolerance, sorted pairs and
    per-gaussian records bit-exact against the reference's collect_kpc output."""
    out = scene.render(cam, L.FilterConfig(tau_r), mode)
    want = ref.render(rh, cam, tau_r, mode, workers=THREADS, collect_kpc=True)
    assert out.stats.n_selected == want["n_selected"], what
    assert out.stats.n_pairs == want["n_pairs"], what
    assert scene.read_pairs().tobytes() == want["pairs"].tobytes(), what
    g = scene.read_gaussians()
    for f in L._LIST_F64 + ("depth", "node"):
        assert getattr(g, f).tobytes() == getattr(want["gaussians"], f).tobytes(), (what, f)
    err = max_abs(out.image.rgb, want["image"])
    assert err <= IMG_TOL, (what, err)
    assert (ref.psnr(out.image.rgb, want["image"]) if err > 0 else np.inf) > PSNR_MIN, what
    return out


@pytest.fixture(scope="module")
def cfg3(L, ref, gpu):
    b = _bench()
    tree = L.build_synthetic_tree(**b.TREE)
    rh = ref.tree_from(tree)
    cams = b.flythrough(L)
    scene = L.GpuScene(tree)
    for cam in cams[::10]:  # size the pair buffer on the path (as the bench does)
        scene.render(cam, L.FilterConfig(b.TAU_R), L.ShrinkMode.three_sigma())
    yield b, tree, rh, cams, scene
    scene.close()
    ref.free_tree(rh)


def test_cfg3_bench_frames_async_and_batch(L, ref, cfg3):
    """The frames the driver's `bench.py --steps 20` times (strided over the whole
    300-frame path), through render_async (4 in flight) and render_batch: every image
    against the reference renderer's; then the same frames with the TMA-staged blend
    kernels (LODGS_RENDER_BLEND_TMA / _GATHER4) and the round-1 default
    k_blend_wsp (LODGS_RENDER_BLEND_WSP, byte-identical to the default k_blend_cpa) against
    the same images."""
    b, tree, rh, cams, scene = cfg3
    from paper_2603_23891_b200.sharding import strided_frames

    idx = strided_frames(len(cams), 0, 1, 20)
    frames = [cams[i] for i in idx]
    mode = L.ShrinkMode.three_sigma()
    a_imgs = _async_frames(L, scene, frames, b.TAU_R, mode)
    b_imgs, b_stats = _batch_frames(L, scene, frames, b.TAU_R, mode)
    worst = 0.0
    wants = []
    for i, cam, ai, bi, st in zip(idx, frames, a_imgs, b_imgs, b_stats):
        want, err, _ = _compare(ref, rh, cam, b.TAU_R, mode, bi, st, f"batch frame {i}")
        assert ai.tobytes() == bi.tobytes(), f"async frame {i} differs from the batch frame"
        worst = max(worst, err)
        wants.append(want)
    print(f"cfg3 bench frames: worst max-abs {worst:.3g}")
    for k in ("tma", "gather4", "wsp"):
        imgs = _async_frames(L, scene, frames, b.TAU_R, mode, blend_kernel=k)
        for i, cam, im, want, bi in zip(idx, frames, imgs, wants, b_imgs):
            _compare(ref, rh, cam, b.TAU_R, mode, im, None, f"{k} frame {i}", want=want)
            if k == "wsp":  # k_blend_cpa's means and sample order: the same bytes
                assert im.tobytes() == bi.tobytes(), f"wsp frame {i} differs from cpa"


def test_sync_render_pinned_bands(L, ref, cfg3):
    """A synchronous render into pinned host memory blends in four horizontal bands and
    copies each band while the next one blends: the 20 bench frames equal
    the pageable-memory renders (one blend, one copy) byte for byte, with four more
    launches; short images (2 and 3 tile rows) and stage timing (no bands) too."""
    b, tree, rh, cams, scene = cfg3
    from paper_2603_23891_b200.sharding import strided_frames

    mode = L.ShrinkMode.three_sigma()
    with L.PinnedImage(1920, 1080) as pin:
        for i in strided_frames(len(cams), 0, 1, 20):
            want = scene.render(cams[i], L.FilterConfig(b.TAU_R), mode)
            got = scene.render(cams[i], L.FilterConfig(b.TAU_R), mode, image_out=pin.rgb)
            assert got.stats.kernel_launches == want.stats.kernel_launches + 4, i
            assert pin.rgb.tobytes() == want.image.rgb.tobytes(), f"frame {i}"
        t = scene.render(cams[150], L.FilterConfig(b.TAU_R), mode,
                         L.RenderOptions(stage_timing=True), image_out=pin.rgb)
        assert t.stats.kernel_launches == want.stats.kernel_launches  # no bands when timed
    for w, h, bands in ((640, 40, 3), (640, 17, 2)):
        cam = topdown_camera(w, h, 300.0, 60.0)
        want = scene.render(cam, L.FilterConfig(b.TAU_R), mode)
        with L.PinnedImage(w, h) as pin:
            got = scene.render(cam, L.FilterConfig(b.TAU_R), mode, image_out=pin.rgb)
            assert got.stats.kernel_launches == want.stats.kernel_launches + bands, (w, h)
            assert pin.rgb.tobytes() == want.image.rgb.tobytes(), (w, h)


def test_cfg3_altitudes_and_oblique_keyframes(L, ref, cfg3):
    """Top-down frames at altitudes 400 / 200 / 140 and the two oblique keyframes
    (260 and 140), synchronous production renders: pairs and BlendList bit-exact,
    image within tolerance."""
    b, tree, rh, cams, scene = cfg3
    mode = L.ShrinkMode.three_sigma()
    keys = b.keyframes(L)
    views = [("alt400", topdown_camera(1920, 1080, 1000.0, 400.0)),
             ("alt200", topdown_camera(1920, 1080, 1000.0, 200.0)),
             ("alt140", topdown_camera(1920, 1080, 1000.0, 140.0)),
             ("oblique260", keys[1]), ("oblique140", keys[3])]
    for name, cam in views:
        _sync_check(L, ref, rh, scene, cam, b.TAU_R, mode, name)


def test_cfg1_production(L, ref, gpu):
    """cfg 1 (99,937 nodes, 800x600, fx=100, z=12) through all three entry points."""
    tree = L.build_synthetic_tree(nx=37, ny=37, seed=1, depth=2, build_seed=7)
    rh = ref.tree_from(tree)
    cam = ref.front_camera(800, 600, 100.0)
    cam.translation = (0, 0, 12)
    cams = [cam]
    for dx in (0.5, -1.0, 1.5):  # a few neighbours of the test camera
        c = ref.front_camera(800, 600, 100.0)
        c.translation = (dx, -dx / 2, 12.0 + dx)
        cams.append(c)
    mode = L.ShrinkMode.three_sigma()
    try:
        with L.GpuScene(tree) as s:
            _sync_check(L, ref, rh, s, cam, 3.0, mode, "cfg1 sync")
            a = _async_frames(L, s, cams, 3.0, mode)
            bi, st = _batch_frames(L, s, cams, 3.0, mode)
            for k, c in enumerate(cams):
                _compare(ref, rh, c, 3.0, mode, bi[k], st[k], f"cfg1 batch {k}")
                assert a[k].tobytes() == bi[k].tobytes()
    finally:
        ref.free_tree(rh)


def test_cfg2_adaptive_calibrated(L, ref, gpu):
    """cfg 2 (1,007,370 nodes, 1080p, altitude 50..60) with GTC shrinking on: tau from
    the device calibration at lambda_G = 0.2 (bit-exact with the reference's
    calibrate, test_gpu_parity), then adaptive production frames against the
    reference renderer at the same tau -- radii, pairs and images at ~10^6 gaussians
    per frame (the CUDA-log vs glibc-log exposure of effective_radius)."""
    b = _bench()
    tree = L.build_synthetic_tree(nx=41, ny=42, seed=1, depth=3, build_seed=7)
    rh = ref.tree_from(tree)
    keys = []
    for eye, target in (((0.0, 0.0, 60.0), (0.0, 0.0001, 0.0)),
                        ((5.0, -3.0, 50.0), (5.0, -2.9999, 0.0))):  # tools/workloads.py cfg2
        R, t = b.look_at(eye, target)
        keys.append(L.Camera(1920, 1080, 1000.0, 1000.0, 960.0, 540.0, R, t))
    cams = L.sample_camera_path(keys, [11])
    try:
        with L.GpuScene(tree) as s:
            rep = s.calibrate(cams[:: 3][:4], 0.2, L.FilterConfig(3.0))
            assert 0.0 < rep.tau < 1.0
            for tau in (rep.tau, 0.02):  # the calibrated tau and a gentle one
                mode = L.ShrinkMode.adaptive(tau)
                _sync_check(L, ref, rh, s, cams[0], 3.0, mode, f"cfg2 adaptive {tau}")
                bi, st = _batch_frames(L, s, cams, 3.0, mode)
                for k, c in enumerate(cams):
                    _compare(ref, rh, c, 3.0, mode, bi[k], st[k], f"cfg2 adaptive {tau} #{k}")
            mode = L.ShrinkMode.three_sigma()
            _sync_check(L, ref, rh, s, cams[-1], 3.0, mode, "cfg2 three-sigma")
    finally:
        ref.free_tree(rh)


def test_cfg4_50m_4k_production(L, ref, gpu):
    """cfg 4 (50,142,872 nodes, 3840x2160, fx = 2000): production renders at altitude
    400 and 110 (23M selected, 40M pairs, buckets into the big-bucket sort), three-sigma
    and adaptive at the device-calibrated tau; pairs bit-exact, images within
    tolerance, and the altitude-110 frame again through render_async."""
    tree = L.build_synthetic_tree(nx=103, ny=104, seed=1, depth=4, build_seed=7)
    assert tree.node_count() == 50142872
    rh = ref.tree_from(tree)
    try:
        with L.GpuScene(tree) as s:
            hi = topdown_camera(3840, 2160, 2000.0, 400.0)
            lo = topdown_camera(3840, 2160, 2000.0, 110.0)
            mode = L.ShrinkMode.three_sigma()
            _sync_check(L, ref, rh, s, hi, 3.0, mode, "cfg4 alt400")
            out = _sync_check(L, ref, rh, s, lo, 3.0, mode, "cfg4 alt110")
            assert out.stats.big_tiles > 0  # the big-bucket sort ran
            a = _async_frames(L, s, [hi, lo], 3.0, mode)
            assert a[1].tobytes() == out.image.rgb.tobytes()
            # the synchronous render into pinned memory: 4K, the 16-stage blend, in bands
            with L.PinnedImage(3840, 2160) as pin:
                pb = s.render(lo, L.FilterConfig(3.0), mode, image_out=pin.rgb)
                assert pb.stats.kernel_launches == out.stats.kernel_launches + 4
                assert pin.rgb.tobytes() == out.image.rgb.tobytes()
            # the multi-view filter on the 50M tree (groups of four over two context sets)
            s.set_inflight(8)
            v = _views(L, s, [hi, lo, hi, lo, lo], 3.0, mode)
            assert v[1].tobytes() == out.image.rgb.tobytes()
            assert v[4].tobytes() == out.image.rgb.tobytes()
            assert v[0].tobytes() == v[2].tobytes() == a[0].tobytes()
            s.set_inflight(4)
            # tools/workloads.py cfg 4: a 30-frame descent 400 -> 300 -> 110, 4 views
            b = _bench()
            keys = []
            for eye, target in (((0.0, 0.0, 400.0), (0.0, 0.0001, 0.0)),
                                ((20.0, -10.0, 300.0), (20.0, -9.9999, 0.0)),
                                ((-10.0, 15.0, 110.0), (-10.0, 15.0001, 0.0))):
                R, t = b.look_at(eye, target)
                keys.append(L.Camera(3840, 2160, 2000.0, 2000.0, 1920.0, 1080.0, R, t))
            path = L.sample_camera_path(keys, [14, 15])
            rep = s.calibrate(path[::7][:4], 0.2, L.FilterConfig(3.0))
            assert 0.0 < rep.tau < 1.0, rep.tau
            mode = L.ShrinkMode.adaptive(rep.tau)
            _sync_check(L, ref, rh, s, lo, 3.0, mode, f"cfg4 alt110 adaptive {rep.tau}")
    finally:
        ref.free_tree(rh)


def test_rgb8_batch_overflow_regrow(L, ref, gpu):
    """render_batch with 8-bit output where frames overflow the pair buffer: the frame
    is re-rendered and its W*H*3 bytes (not floats) land in the caller's buffer, equal
    to the save_ppm quantisation of the float frame (the overflow path used
    to copy W*H*3 floats into a W*H*3-byte buffer)."""
    tree = L.make_tree(33, 3, 8, 0.5, 3, 3, 3)
    cam = ref.front_camera(1024, 1024, 2000.0)
    cam.translation = (0, 0, 9.0)
    cams = [cam, cam]
    with L.GpuScene(tree) as s:
        # the scene starts with max(4N, 65536) pairs; this close-up needs more, so both
        # batch frames overflow and are re-rendered after the buffer grows
        mem0 = s.memory_bytes()
        guard = 4096
        bufs = [np.full(1024 * 1024 * 3 + guard, 0xAB, np.uint8) for _ in cams]
        st = s.render_batch(cams, L.FilterConfig(1e9), L.ShrinkMode.three_sigma(),
                            L.RenderOptions(output_rgb8=True),
                            host_ptrs=[b.ctypes.data for b in bufs])
        assert s.memory_bytes() > mem0, "the pair buffer did not grow: no overflow exercised"
        full = s.render(cam, L.FilterConfig(1e9), L.ShrinkMode.three_sigma())
        want8 = s.read_image_rgb8(cam)
        for b, one in zip(bufs, st):
            assert (b[-guard:] == 0xAB).all(), "wrote past the 8-bit host buffer"
            assert b[:-guard].tobytes() == want8.tobytes()
            assert one.n_pairs == full.stats.n_pairs


def test_read_image_after_async_then_batch(L, oracle, gpu):
    """read_image after render_async (last frame on a twin context) followed
    by render_batch must return the batch's last frame."""
    tree = L.make_tree(23, 3, 8, 0.5, 4, 4, 2)
    rng = oracle.rng(3)
    cams = [oracle.orbit_camera(rng, 200, 150, 16.0) for _ in range(6)]
    for c in cams:
        c.fx = c.fy = 150.0
    mode = L.ShrinkMode.three_sigma()
    with L.GpuScene(tree) as s:
        p = s.params(L.FilterConfig(4.0), mode, L.RenderOptions())
        for cam in cams[:3]:
            s.render_async(cam, p)
        s.sync()
        s.render_batch(cams[3:], L.FilterConfig(4.0), mode)
        got = s.read_image(cams[-1])
        want = s.render(cams[-1], L.FilterConfig(4.0), mode).image.rgb
        assert got.tobytes() == want.tobytes()


def test_large_tile_grid_2048x1536(L, oracle, gpu):
    """A 2048x1536 frame (128x96 = 12,288 tiles: the largest shared-memory tile
    histogram in K3/K4, which needs the >48 KB dynamic shared-memory opt-in)."""
    tree = L.make_tree(41, 3, 8, 0.5, 4, 4, 2)
    cam = oracle.front_camera(2048, 1536, 900.0)
    cam.translation = (0.0, 0.0, 18.0)
    mode = L.ShrinkMode.three_sigma()
    want = oracle.render(tree, cam, 3.0, mode)
    with L.GpuScene(tree) as s:
        out = s.render(cam, L.FilterConfig(3.0), mode)
    assert out.stats.n_pairs == want["n_pairs"] and out.stats.n_pairs > 0
    assert max_abs(out.image.rgb, want["image"]) <= IMG_TOL
