"""SURVEY.md 8(f) row 4 on the device: psnr / ssim (metrics.cpp:121-192), the
8-bit output of save_ppm (image.cpp:12-28), on-device reference comparison,
and render(..., RenderOptions{filter_mode = serial}) (rasterizer.hpp:96-104).

The metric sums are re-associated on the device (per-CTA trees), so psnr/ssim
are compared with the compiled reference to 1e-12 relative; the 8-bit bytes
are bit-exact.
"""
import math

import numpy as np
import pytest

from helpers import topdown_camera

pytestmark = pytest.mark.gpu

METRIC_RTOL = 1e-12


def _rgb8_restated(img):
    """image.cpp:19-22 in float32: clamp, v * 255.f + 0.5f, floor."""
    x = np.clip(np.asarray(img, np.float32), np.float32(0.0), np.float32(1.0))
    return np.floor(x * np.float32(255.0) + np.float32(0.5)).astype(np.uint8)


def test_psnr_ssim_match_reference(L, ref, gpu):
    rng = np.random.default_rng(3)
    for (h, w, noise) in ((11, 11, 0.1), (40, 53, 0.01), (120, 97, 0.3), (64, 64, 1e-4)):
        a = rng.random((h, w, 3), dtype=np.float32)
        b = np.clip(a + rng.normal(0, noise, a.shape).astype(np.float32), 0, 1)
        p, q = L.psnr(a, b), L.ssim(a, b)
        pr, qr = ref.psnr(a, b), ref.ssim(a, b)
        assert abs(p - pr) <= METRIC_RTOL * abs(pr), (h, w, p, pr)
        assert abs(q - qr) <= METRIC_RTOL * max(1.0, abs(qr)), (h, w, q, qr)
    assert L.psnr(a, a) == math.inf
    assert abs(L.ssim(a, a) - 1.0) <= 1e-12


def test_metric_errors(L, gpu):
    a = np.zeros((20, 20, 3), np.float32)
    with pytest.raises(L.ValidationError):
        L.psnr(a, np.zeros((20, 21, 3), np.float32))
    with pytest.raises(L.ValidationError):
        L.ssim(np.zeros((10, 30, 3), np.float32), np.zeros((10, 30, 3), np.float32))


def test_rendered_frames_metrics_and_rgb8(L, ref, gpu):
    """A three-sigma frame is the reference of a shrunk frame (bench.cpp's
    psnr_vs_ref / ssim_vs_ref); device comparison == host metric == the
    compiled reference; 8-bit readback == the save_ppm quantisation."""
    tree = L.build_synthetic_tree(nx=37, ny=37, seed=1, depth=2, build_seed=7)
    cam = topdown_camera(320, 240, 150.0, 30.0)
    with L.GpuScene(tree) as s:
        a = s.render(cam, L.FilterConfig(3.0), L.ShrinkMode.three_sigma()).image.rgb.copy()
        b8a = s.read_image_rgb8(cam)
        assert np.array_equal(b8a, _rgb8_restated(a))
        s.set_reference_image()
        b = s.render(cam, L.FilterConfig(3.0), L.ShrinkMode.adaptive(0.3)).image.rgb.copy()
        p, q = s.compare_reference()
        pr, qr = ref.psnr(b, a), ref.ssim(b, a)
        assert abs(p - pr) <= METRIC_RTOL * abs(pr) and abs(q - qr) <= METRIC_RTOL
        assert abs(L.psnr(b, a) - pr) <= METRIC_RTOL * abs(pr)
        assert np.array_equal(s.read_image_rgb8(cam), _rgb8_restated(b))
        # 4x the pixels: a resolution change invalidates the stored reference
        cam2 = topdown_camera(640, 480, 300.0, 30.0)
        s.render(cam2, L.FilterConfig(3.0), L.ShrinkMode.three_sigma())
        with pytest.raises(L.ValidationError):
            s.compare_reference()


def test_render_filter_serial_mode(L, oracle, ref, gpu):
    """RenderOptions::filter_mode = serial: the frame's filter is the level-wise
    one; image, pairs and selection equal the parallel frame (the generated
    trees nest child spheres in their parents'), passes = barriers = the
    reference renderer's serial counts."""
    tree = L.build_synthetic_tree(nx=37, ny=37, seed=1, depth=2, build_seed=7)
    cam = oracle.front_camera(800, 600, 100.0)
    cam.translation = (0, 0, 12)
    h = ref.tree_from(tree)
    try:
        want = ref.render(h, cam, 3.0, L.ShrinkMode.three_sigma(), filter_mode=1)  # serial
    finally:
        ref.free_tree(h)
    with L.GpuScene(tree) as s:
        ser = s.render(cam, L.FilterConfig(3.0), L.ShrinkMode.three_sigma(),
                       L.RenderOptions(filter_mode="serial", exact_blend=True))
        par = s.render(cam, L.FilterConfig(3.0), L.ShrinkMode.three_sigma(),
                       L.RenderOptions(exact_blend=True))
    assert ser.image.rgb.tobytes() == par.image.rgb.tobytes()
    assert ser.image.rgb.tobytes() == want["image"].tobytes()
    assert ser.stats.n_pairs == par.stats.n_pairs == want["n_pairs"]
    assert ser.stats.filter_passes == want["passes"] == 3
    assert ser.stats.filter_barriers == want["barriers"]
    assert par.stats.filter_passes == 2
    with pytest.raises(L.ValidationError):
        L.GpuScene.params(L.FilterConfig(3.0), L.ShrinkMode.three_sigma(),
                          L.RenderOptions(filter_mode="oracle"))


def test_render_batch_rgb8_output(L, oracle, gpu):
    """render_batch with LODGS_RENDER_OUTPUT_RGB8: every host image is the
    save_ppm quantisation of the frame's f32 image."""
    tree = L.make_tree(21, 3, 8, 0.5, 3, 3, 2)
    rng = oracle.rng(5)
    cams = [oracle.orbit_camera(rng, 200, 150, 14.0) for _ in range(4)]
    for c in cams:
        c.fx = c.fy = 150.0
    b8 = [np.zeros((150, 200, 3), np.uint8) for _ in cams]
    with L.GpuScene(tree) as s:
        s.render_batch(cams, L.FilterConfig(4.0), L.ShrinkMode.three_sigma(),
                       L.RenderOptions(output_rgb8=True), host_ptrs=[b.ctypes.data for b in b8])
        for cam, b in zip(cams, b8):
            f = s.render(cam, L.FilterConfig(4.0), L.ShrinkMode.three_sigma()).image.rgb
            assert np.array_equal(b, _rgb8_restated(f))
