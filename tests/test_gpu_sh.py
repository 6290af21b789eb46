"""View-dependent colour, spherical harmonics of degree 1..3 (lodgs_gpu_scene_set_sh):
the extension behind BASELINE.json configs[1] ("SH deg 3").

The reference is SH0-only (scene.hpp:15-24), so these colours have no
reference to match: parity is pinned where it can be -- with every coefficient zero a
frame is the SH0 frame bit for bit (image, pairs, BlendList) -- and otherwise against
the numpy restatement below of the device evaluation (the 3DGS real SH basis on top of
the node's SH0 colour, FP64, the device's operation order: bit-exact after the f32
rounding the BlendList readback applies).  Fast and exact blends of SH frames agree
within the north-star tolerance.
"""
import numpy as np
import pytest

from helpers import max_abs, topdown_camera

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-3

C1 = 0.4886025119029199
C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
      0.5462742152960396)
C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
      -0.4570457994644658, 1.445305721320277, -0.5900435899266435)


def basis(k, x, y, z):
    """preprocess.cu sh_basis, left to right as C++ evaluates it."""
    xx, yy, zz = x * x, y * y, z * z
    return [
        lambda: -C1 * y, lambda: C1 * z, lambda: -C1 * x,
        lambda: C2[0] * (x * y), lambda: C2[1] * (y * z), lambda: C2[2] * (2.0 * zz - xx - yy),
        lambda: C2[3] * (x * z), lambda: C2[4] * (xx - yy),
        lambda: C3[0] * y * (3.0 * xx - yy), lambda: C3[1] * (x * y) * z,
        lambda: C3[2] * y * (4.0 * zz - xx - yy), lambda: C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy),
        lambda: C3[4] * x * (4.0 * zz - xx - yy), lambda: C3[5] * z * (xx - yy),
        lambda: C3[6] * x * (xx - 3.0 * yy),
    ][k]()


def sh_colours(tree, cam, nodes, sh):
    """k_sh_colour restated in numpy float64 (vectorised over nodes; elementwise IEEE
    operations in the kernel's order, no FMA)."""
    R = np.asarray(cam.rotation, np.float64)
    t = np.asarray(cam.translation, np.float64)
    cx = -((R[0] * t[0] + R[3] * t[1]) + R[6] * t[2])
    cy = -((R[1] * t[0] + R[4] * t[1]) + R[7] * t[2])
    cz = -((R[2] * t[0] + R[5] * t[1]) + R[8] * t[2])
    dx = tree.mean_x[nodes].astype(np.float64) - cx
    dy = tree.mean_y[nodes].astype(np.float64) - cy
    dz = tree.mean_z[nodes].astype(np.float64) - cz
    inv = 1.0 / np.sqrt((dx * dx + dy * dy) + dz * dz)
    x, y, z = dx * inv, dy * inv, dz * inv
    cols = [tree.color_r[nodes].astype(np.float64), tree.color_g[nodes].astype(np.float64),
            tree.color_b[nodes].astype(np.float64)]
    c = sh[nodes].astype(np.float64)
    for k in range(sh.shape[1]):
        Y = basis(k, x, y, z)
        for ch in range(3):
            cols[ch] = cols[ch] + Y * c[:, k, ch]
    return [np.where(v < 0.0, 0.0, v) for v in cols]


@pytest.fixture(scope="module")
def scene_sh(L, gpu):
    tree = L.build_synthetic_tree(nx=9, ny=9, seed=1, depth=3, build_seed=7)
    with L.GpuScene(tree) as s:
        yield tree, s


def _frame(L, s, cam, **opts):
    return s.render(cam, L.FilterConfig(3.0), L.ShrinkMode.three_sigma(), L.RenderOptions(**opts))


def _cams(L):
    return [topdown_camera(640, 480, 500.0, 30.0, 0.5, -0.3),
            L.Camera(640, 480, 400.0, 400.0, 320.0, 240.0,
                     (0.8, 0.6, 0.0, 0.36, -0.48, -0.8, -0.48, 0.64, -0.6), (0.5, 1.0, 25.0))]


def test_zero_coefficients_equal_sh0(L, scene_sh):
    """Degree 1..3 with all coefficients zero: every frame is the SH0 frame, bit for bit
    (exact and fast images, sorted pairs, every BlendList field)."""
    tree, s = scene_sh
    n = tree.node_count()
    for cam in _cams(L):
        s.set_sh(0)
        base = _frame(L, s, cam, collect_kpc=True)
        base_fast = _frame(L, s, cam).image.rgb.copy()
        for deg in (1, 2, 3):
            s.set_sh(deg, np.zeros((n, (deg + 1) ** 2 - 1, 3), np.float32))
            out = _frame(L, s, cam, collect_kpc=True)
            assert out.image.rgb.tobytes() == base.image.rgb.tobytes(), deg
            assert out.pairs.tobytes() == base.pairs.tobytes(), deg
            for f in L._LIST_F64 + ("depth", "node"):
                assert getattr(out.gaussians, f).tobytes() == getattr(base.gaussians, f).tobytes(), (deg, f)
            assert _frame(L, s, cam).image.rgb.tobytes() == base_fast.tobytes(), deg
    s.set_sh(0)


def test_sh_colours_match_restatement(L, scene_sh):
    """Random coefficients, degrees 1..3, two views: the BlendList colours equal the
    numpy restatement rounded to f32; geometry is unchanged; the fast image is within
    the tolerance of the exact (FP64-colour) image and differs from the SH0 image."""
    tree, s = scene_sh
    n = tree.node_count()
    rng = np.random.default_rng(3)
    for deg in (1, 2, 3):
        sh = rng.normal(0.0, 0.2, (n, (deg + 1) ** 2 - 1, 3)).astype(np.float32)
        for cam in _cams(L):
            s.set_sh(0)
            sh0 = _frame(L, s, cam, collect_kpc=True)
            s.set_sh(deg, sh)
            out = _frame(L, s, cam, collect_kpc=True)
            g = out.gaussians
            want = sh_colours(tree, cam, np.asarray(g.node, np.int64), sh)
            for ch, f in enumerate(("col_r", "col_g", "col_b")):
                got = np.asarray(getattr(g, f))
                assert got.tobytes() == want[ch].astype(np.float32).astype(np.float64).tobytes(), (deg, f)
            for f in ("mean_x", "mean_y", "conic_a", "conic_b", "conic_c", "opacity", "radius",
                      "depth", "node"):
                assert getattr(g, f).tobytes() == getattr(sh0.gaussians, f).tobytes(), (deg, f)
            assert out.pairs.tobytes() == sh0.pairs.tobytes()
            fast = _frame(L, s, cam).image.rgb
            assert max_abs(fast, out.image.rgb) <= IMG_TOL, deg
            assert max_abs(out.image.rgb, sh0.image.rgb) > 1e-2, deg  # the colours did change
    s.set_sh(0)


def test_sh_frames_in_flight(L, scene_sh):
    """SH frames through render_batch (pipelined over the four in-flight contexts) and
    render_async equal the synchronous renders."""
    tree, s = scene_sh
    n = tree.node_count()
    sh = np.random.default_rng(4).normal(0.0, 0.2, (n, 15, 3)).astype(np.float32)
    s.set_sh(3, sh)
    cams = [topdown_camera(640, 480, 500.0, 20.0 + 3 * i, 0.1 * i, 0.0) for i in range(6)]
    want = [_frame(L, s, c).image.rgb.copy() for c in cams]
    imgs = [np.empty((c.height, c.width, 3), np.float32) for c in cams]
    s.render_batch(cams, L.FilterConfig(3.0), L.ShrinkMode.three_sigma(),
                   host_ptrs=[im.ctypes.data for im in imgs])
    for w, im in zip(want, imgs):
        assert im.tobytes() == w.tobytes()
    p = s.params(L.FilterConfig(3.0), L.ShrinkMode.three_sigma(), L.RenderOptions())
    for c, w in zip(cams, want):
        s.render_async(c, p)
        s.sync()
        assert s.read_image(c).tobytes() == w.tobytes()
    # the multi-view filter: SH colours on every context
    s.set_inflight(8)
    vimgs = [np.empty((c.height, c.width, 3), np.float32) for c in cams]
    s.render_views_async(cams, p, host_ptrs=[im.ctypes.data for im in vimgs])
    s.sync()
    for w, im in zip(want, vimgs):
        assert im.tobytes() == w.tobytes()
    s.set_inflight(4)
    s.set_sh(0)


def test_set_sh_validation(L, scene_sh):
    tree, s = scene_sh
    n = tree.node_count()
    with pytest.raises(L.ValidationError):
        s.set_sh(4, np.zeros((n, 24, 3), np.float32))
    with pytest.raises(L.ValidationError):
        s.set_sh(3, np.zeros((n, 8, 3), np.float32))  # degree 2's shape
    with pytest.raises(L.ValidationError):
        s.set_sh(1, np.zeros((n - 1, 3, 3), np.float32))  # one row per node
    bad = np.zeros((n, 3, 3), np.float32)
    bad[n // 2, 1, 2] = np.nan
    with pytest.raises(L.ValidationError):
        s.set_sh(1, bad)
    s.set_sh(0)
