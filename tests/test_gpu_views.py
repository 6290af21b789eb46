"""The multi-view filter (lodgs_gpu_render_views_async, SURVEY.md 8(e)'s option): the
LoD filter of up to four consecutive frames in one pass over the node arrays.  Every
frame must equal its single-view render bit for bit -- image, selected list, counters
-- for any group size, any number of frames in flight, and the large-tree compaction
path (> 2048 compaction tiles, k_tile_prefix)."""
import numpy as np
import pytest

from helpers import topdown_camera

pytestmark = pytest.mark.gpu


def _views_frames(L, scene, cams, tau_r=3.0):
    imgs = [np.empty((c.height, c.width, 3), np.float32) for c in cams]
    p = scene.params(L.FilterConfig(tau_r), L.ShrinkMode.three_sigma(), L.RenderOptions())
    scene.take_totals()
    scene.render_views_async(cams, p, host_ptrs=[im.ctypes.data for im in imgs])
    scene.sync()
    return imgs, scene.take_totals()


def _sync_frames(L, scene, cams, tau_r=3.0):
    out, sel, pairs = [], 0, 0
    for c in cams:
        r = scene.render(c, L.FilterConfig(tau_r), L.ShrinkMode.three_sigma())
        out.append(r.image.rgb.copy())
        sel += r.stats.n_selected
        pairs += r.stats.n_pairs
    return out, sel, pairs


@pytest.fixture(scope="module")
def city(L, gpu):
    import bench

    tree = L.build_synthetic_tree(**bench.TREE)
    cams = bench.flythrough(L)
    with L.GpuScene(tree) as s:
        yield tree, cams, s


def test_views_bench_frames(L, city):
    """The driver's 20 strided cfg-3 bench frames through render_views_async (groups of
    four, eight frames in flight): every image equals the synchronous render's, and the
    summed selected / pair counts equal too."""
    from paper_2603_23891_b200.sharding import strided_frames

    tree, cams, s = city
    s.set_inflight(8)
    frames = [cams[i] for i in strided_frames(len(cams), 0, 1, 20)]
    want, sel, pairs = _sync_frames(L, s, frames)
    got, (nf, gsel, gpairs) = _views_frames(L, s, frames)
    assert nf == len(frames) and gsel == sel and gpairs == pairs
    for i, (w, g) in enumerate(zip(want, got)):
        assert g.tobytes() == w.tobytes(), f"frame {i}"
    s.set_inflight(4)


@pytest.mark.parametrize("inflight", [3, 4, 6, 8])
def test_views_group_sizes(L, city, inflight):
    """1..9 frames with 3 (per-frame fallback), 4, 6 or 8 frames in flight (groups of
    2, 3, 4 views over two context sets, ragged last groups): every image and the
    summed counters equal the single-view renders'."""
    tree, cams, s = city
    s.set_inflight(inflight)
    for n in (1, 2, 3, 5, 9):
        frames = [cams[(37 * k + 11 * n) % len(cams)] for k in range(n)]
        want, sel, pairs = _sync_frames(L, s, frames)
        got, (nf, gsel, gpairs) = _views_frames(L, s, frames)
        assert (nf, gsel, gpairs) == (n, sel, pairs), (inflight, n)
        for i, (w, g) in enumerate(zip(want, got)):
            assert g.tobytes() == w.tobytes(), (inflight, n, i)
    s.set_inflight(4)


def test_views_large_tree_prefix_path(L, gpu):
    """A 20M-node tree (2,500+ compaction tiles: the per-view prefix scan) and mixed
    altitudes, five frames in one call."""
    tree = L.build_synthetic_tree(nx=185, ny=185, seed=1, depth=3, build_seed=7)
    assert tree.node_count() > 2048 * 8192
    cams = [topdown_camera(1920, 1080, 1000.0, a, 3.0 * k, -2.0 * k)
            for k, a in enumerate((400.0, 250.0, 180.0, 140.0, 300.0))]
    with L.GpuScene(tree) as s:
        s.set_inflight(8)
        want, sel, pairs = _sync_frames(L, s, cams)
        got, (nf, gsel, gpairs) = _views_frames(L, s, cams)
        assert (nf, gsel, gpairs) == (len(cams), sel, pairs)
        for i, (w, g) in enumerate(zip(want, got)):
            assert g.tobytes() == w.tobytes(), i


def test_views_fall_back_per_frame(L, city):
    """Per-frame-only flags (stage timing) take the per-frame path: same images."""
    tree, cams, s = city
    frames = cams[100:103]
    want, _, _ = _sync_frames(L, s, frames)
    imgs = [np.empty((c.height, c.width, 3), np.float32) for c in frames]
    p = s.params(L.FilterConfig(3.0), L.ShrinkMode.three_sigma(), L.RenderOptions(stage_timing=True))
    s.render_views_async(frames, p, host_ptrs=[im.ctypes.data for im in imgs])
    s.sync()
    for w, g in zip(want, imgs):
        assert g.tobytes() == w.tobytes()


def test_views_adaptive_and_rgb8(L, city):
    """Adaptive shrinking (the filter is mode-independent, K3 is not) and 8-bit host images
    (LODGS_RENDER_OUTPUT_RGB8) through render_views_async: equal to the per-frame path."""
    from paper_2603_23891_b200.sharding import strided_frames

    tree, cams, s = city
    s.set_inflight(8)
    frames = [cams[i] for i in strided_frames(len(cams), 0, 1, 8)]
    mode = L.ShrinkMode.adaptive(0.05)
    want = [s.render(c, L.FilterConfig(3.0), mode).image.rgb.copy() for c in frames]
    imgs = [np.empty((c.height, c.width, 3), np.float32) for c in frames]
    p = s.params(L.FilterConfig(3.0), mode, L.RenderOptions())
    s.render_views_async(frames, p, host_ptrs=[im.ctypes.data for im in imgs])
    s.sync()
    for i, (w, g) in enumerate(zip(want, imgs)):
        assert g.tobytes() == w.tobytes(), f"adaptive frame {i}"
    three = L.ShrinkMode.three_sigma()
    want8 = []
    for c in frames:
        s.render(c, L.FilterConfig(3.0), three)
        want8.append(s.read_image_rgb8(c))
    b8 = [np.empty((c.height, c.width, 3), np.uint8) for c in frames]
    p8 = s.params(L.FilterConfig(3.0), three, L.RenderOptions(output_rgb8=True))
    s.render_views_async(frames, p8, host_ptrs=[im.ctypes.data for im in b8])
    s.sync()
    for i, (w, g) in enumerate(zip(want8, b8)):
        assert g.tobytes() == w.tobytes(), f"rgb8 frame {i}"
    s.set_inflight(4)
