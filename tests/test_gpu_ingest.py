"""SURVEY.md 8(f) row 2 on the device: LDGS v1 scene files loaded straight into
a GpuScene (scene_io.cpp:90-116, 213-226) and validate_tree's per-node rules
(scene.cpp:122-162) run by a kernel at scene creation.

Checked against the reference itself (oracle/_ref/ref_ldgs_tool runs the
reference's save_scene / load_scene natively) and against the host validator
that the CPU suite pins to the reference.
"""
import os

import numpy as np
import pytest

from helpers import REF_LDGS_TOOL, ref_ldgs, topdown_camera, write_ldgs

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(REF_LDGS_TOOL), reason="oracle/_ref not built")]


def _same_scene(L, a, b, cam, tau_r=3.0):
    fa = a.filter(cam, L.FilterConfig(tau_r)).selected
    fb = b.filter(cam, L.FilterConfig(tau_r)).selected
    assert np.array_equal(fa, fb)
    opts = L.RenderOptions(exact_blend=True)
    ia = a.render(cam, L.FilterConfig(tau_r), L.ShrinkMode.three_sigma(), opts).image.rgb
    ib = b.render(cam, L.FilterConfig(tau_r), L.ShrinkMode.three_sigma(), opts).image.rgb
    assert ia.tobytes() == ib.tobytes()


def test_load_reference_written_scene(L, gpu, tmp_path):
    path = tmp_path / "ref.ldgs"
    assert ref_ldgs("save", path, 21, 19, 3, 3, 11) == "SAVED"
    tree = L.build_synthetic_tree(nx=21, ny=19, seed=3, depth=3, build_seed=11)
    tm = np.zeros(3)
    with L.GpuScene.load(str(path), timing_ms=tm) as s, L.GpuScene(tree) as t:
        assert s.tree.node_count() == tree.node_count()
        assert np.array_equal(s.tree.level_offsets, tree.level_offsets)
        assert abs(s.tree.shrink_factor - tree.shrink_factor) == 0
        for alt in (30.0, 80.0):
            _same_scene(L, s, t, topdown_camera(640, 480, 500.0, alt))
    assert (tm >= 0).all()


def test_load_errors_match_reference(L, gpu, tmp_path):
    """Missing file -> IoError; bad magic, unsupported version and truncation
    in every section -> FormatError with the reference's message; the
    reference tool agrees on every case."""
    tree = L.make_tree(5, 3, 8, 0.5, 3, 3)
    good = tmp_path / "good.ldgs"
    write_ldgs(tree, good)
    data = good.read_bytes()
    n = tree.node_count()
    cases = {"missing": None, "magic": b"LDGX" + data[4:], "version": data[:4] + b"\x02\x00\x00\x00" + data[8:]}
    sections = (("means", 12 * n), ("scales", 12 * n), ("quaternions", 16 * n), ("opacity", 4 * n),
                ("colors", 12 * n), ("parents", 4 * n), ("leaf flags", n),
                ("level offsets", 4 * len(tree.level_offsets)))
    off = 20
    for what, nb in sections:
        cases["trunc " + what] = data[: off + nb // 2]
        off += nb
    cases["trunc header"] = data[:14]
    for name, blob in cases.items():
        p = tmp_path / f"{name.replace(' ', '_')}.ldgs"
        if blob is not None:
            p.write_bytes(blob)
        want = ref_ldgs("load", p)
        assert want.startswith("ERR"), (name, want)
        kind, msg = want.split(" ", 2)[1:]
        exc = L.IoError if kind == "IoError" else L.ValidationError
        with pytest.raises(exc) as ei:
            L.GpuScene.load(str(p))
        if kind == "FormatError":
            assert msg in str(ei.value), (name, msg, str(ei.value))


def test_load_rejects_invalid_trees_like_the_reference(L, gpu, tmp_path):
    """Per-node rule violations in a file: the device validator refuses the
    scene (ValidationError) exactly when the reference's load_scene does."""
    for case in range(6):
        tree = L.make_tree(40 + case, 2, 4, 0.5, 3, 3)
        i = 7 + 3 * case
        if case == 0:
            tree.mean_x[i] = np.nan
        elif case == 1:
            tree.quat_w[i] = 2.0
        elif case == 2:
            tree.leaf[i] = 1 - tree.leaf[i]
        elif case == 3:
            tree.color_b[i] = -0.5
        elif case == 4:
            tree.parent[i] = L.ROOT_PARENT
        # case 5: valid
        p = tmp_path / f"c{case}.ldgs"
        write_ldgs(tree, p)
        want = ref_ldgs("load", p)
        if case == 5:
            assert want.startswith("OK")
            with L.GpuScene.load(str(p)) as s:
                assert s.tree.node_count() == tree.node_count()
        else:
            assert want.startswith("ERR ValidationError"), want
            with pytest.raises(L.ValidationError):
                L.GpuScene.load(str(p))


def test_device_validator_matches_host_validator(L, oracle, gpu):
    """acceptance.cpp:519-542 (#11) corruptions (plus multi-violation trees):
    scene creation (device per-node rules) raises the same message as the
    host validator (require_valid)."""
    for i in range(60):
        t = L.make_tree(7000 + i, 2, 4, 0.5, 2, 2)
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
        if i % 5 == 0:  # several violations at once: message order and count
            t.opacity[(n + 3) % t.node_count()] = 7.0
            t.scale_z[(n + 11) % t.node_count()] = 0.0
        with pytest.raises(L.ValidationError) as host:
            L.require_valid(t)
        with pytest.raises(L.ValidationError) as dev:
            L.GpuScene(t)
        assert str(dev.value) == str(host.value), i
