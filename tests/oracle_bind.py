"""ctypes bindings to the CPU checkers -- TEST INFRASTRUCTURE ONLY.

* ``Oracle``: oracle/_build/liboracle.so, our plain-C restatement of the
  reference path (oracle/lodgs_oracle.c).
* ``Ref``: oracle/_ref/libref_lodgs.so, the unmodified reference library
  compiled in place from /root/reference (oracle/Makefile) behind a flat shim
  (oracle/ref_shim.cpp).  Optional: present whenever build() ran in a
  container that had /root/reference; it travels to the GPU box as a file.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2603_23891_b200 import lodgs as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libref_lodgs.so")

CameraC = L.CameraC  # identical layout in all three libraries
_FP = C.POINTER(C.c_float)
_DP = C.POINTER(C.c_double)
P = C.c_void_p


class OrcTree(C.Structure):
    _fields_ = [("n", C.c_uint64)] + [(f, _FP) for f in L._FIELDS] + [
        ("parent", C.POINTER(C.c_uint32)),
        ("leaf", C.POINTER(C.c_uint8)),
        ("level_offsets", C.POINTER(C.c_uint32)),
        ("n_levels", C.c_uint32),
    ]


class OrcStats(C.Structure):
    _fields_ = [("n_selected", C.c_uint64), ("n_pairs", C.c_uint64),
                ("n_gaussians", C.c_uint64), ("passes", C.c_int32), ("barriers", C.c_int32)]


class RefStats(C.Structure):
    _fields_ = [("n_selected", C.c_uint64), ("n_pairs", C.c_uint64),
                ("n_gaussians", C.c_uint64), ("passes", C.c_int32), ("barriers", C.c_int32),
                ("t_calc_ms", C.c_double), ("t_sync_ms", C.c_double), ("t_prepr_ms", C.c_double),
                ("t_sort_ms", C.c_double), ("t_alpha_ms", C.c_double)]


def orc_tree(t: L.LoDTree) -> OrcTree:
    o = OrcTree()
    o.n = t.node_count()
    for f in L._FIELDS:
        setattr(o, f, getattr(t, f).ctypes.data_as(_FP))
    o.parent = t.parent.ctypes.data_as(C.POINTER(C.c_uint32))
    o.leaf = t.leaf.ctypes.data_as(C.POINTER(C.c_uint8))
    o.level_offsets = t.level_offsets.ctypes.data_as(C.POINTER(C.c_uint32))
    o.n_levels = t.level_count()
    o._keep = t  # lifetime
    return o


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    """Our C restatement (the parity checker)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run make -C oracle restate")
        lib = C.CDLL(ORACLE_SO)
        lib.orc_rng_sizeof.restype = C.c_size_t
        lib.orc_rng_next_u64.restype = C.c_uint64
        lib.orc_rng_next_u64.argtypes = [P]
        lib.orc_rng_seed.argtypes = [P, C.c_uint64]
        lib.orc_rng_uniform.restype = C.c_double
        lib.orc_rng_uniform.argtypes = [P, C.c_double, C.c_double]
        lib.orc_rng_next_below.restype = C.c_uint64
        lib.orc_rng_next_below.argtypes = [P, C.c_uint64]
        lib.orc_mix_seed.restype = C.c_uint64
        lib.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.orc_front_camera.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.POINTER(CameraC)]
        lib.orc_orbit_camera.argtypes = [P, C.c_uint32, C.c_uint32, C.c_double, C.POINTER(CameraC)]
        lib.orc_camera_geom.argtypes = [C.POINTER(CameraC), _DP]
        lib.orc_mark.argtypes = [_DP, C.POINTER(OrcTree), C.c_uint64, C.c_uint64, C.c_double, P, P, P]
        lib.orc_filter.argtypes = [C.POINTER(OrcTree), C.POINTER(CameraC), C.c_double, C.c_int, P,
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        lib.orc_effective_radius.restype = C.c_double
        lib.orc_effective_radius.argtypes = [C.c_double, C.c_float, C.c_int, C.c_double,
                                             C.POINTER(C.c_int)]
        lib.orc_prepare.argtypes = [C.POINTER(OrcTree), C.POINTER(CameraC), P, C.c_uint64, C.c_int,
                                    C.c_double, C.POINTER(L.BlendListC)]
        lib.orc_bin_count.restype = C.c_uint64
        lib.orc_bin_count.argtypes = [C.POINTER(L.BlendListC), C.c_int, C.c_int]
        lib.orc_bin_to_tiles.restype = C.c_uint64
        lib.orc_bin_to_tiles.argtypes = [C.POINTER(L.BlendListC), C.c_int, C.c_int, P]
        lib.orc_sort_pairs.argtypes = [P, C.c_uint64]
        lib.orc_exp_mx.restype = C.c_double
        lib.orc_exp_mx.argtypes = [C.c_double]
        lib.orc_alpha_blend.argtypes = [P, C.c_uint64, C.POINTER(L.BlendListC), C.c_int, C.c_int,
                                        P, P]
        lib.orc_render.restype = P
        lib.orc_render.argtypes = [C.POINTER(OrcTree), C.POINTER(CameraC), C.c_double, C.c_int,
                                   C.c_double, C.c_int, C.POINTER(C.c_int)]
        lib.orc_render_stats.argtypes = [P, C.POINTER(OrcStats)]
        for fn in ("orc_render_image", "orc_render_pairs", "orc_render_kpc", "orc_render_selected"):
            getattr(lib, fn).restype = P
            getattr(lib, fn).argtypes = [P]
        lib.orc_render_gaussians.argtypes = [P, C.POINTER(L.BlendListC)]
        lib.orc_render_free.argtypes = [P]
        lib.orc_view_gtc.restype = C.c_double
        lib.orc_view_gtc.argtypes = [P, P, C.c_uint64]
        lib.orc_psnr.restype = C.c_double
        lib.orc_psnr.argtypes = [P, P, C.c_uint64]
        self.lib = lib

    # rng
    def rng(self, seed):
        buf = C.create_string_buffer(self.lib.orc_rng_sizeof())
        self.lib.orc_rng_seed(buf, seed)
        return buf

    def front_camera(self, w, h, focal=100.0) -> L.Camera:
        c = CameraC()
        self.lib.orc_front_camera(w, h, focal, C.byref(c))
        return L.Camera.from_c(c)

    def orbit_camera(self, rng, w, h, dist) -> L.Camera:
        c = CameraC()
        self.lib.orc_orbit_camera(rng, w, h, dist, C.byref(c))
        return L.Camera.from_c(c)

    def uniform(self, rng, lo, hi):
        return self.lib.orc_rng_uniform(rng, lo, hi)

    def next_below(self, rng, n):
        return self.lib.orc_rng_next_below(rng, n)

    def camera_geom(self, cam):
        out = np.zeros(44)
        c = cam.to_c()
        self.lib.orc_camera_geom(C.byref(c), out.ctypes.data_as(_DP))
        return out

    def mark(self, tree, cam, tau_r, begin=0, end=None):
        n = tree.node_count()
        end = n if end is None else end
        vis = np.zeros(n, np.uint8)
        q = np.zeros(n, np.uint8)
        r = np.zeros(n, np.float64)
        g = self.camera_geom(cam)
        t = orc_tree(tree)
        self.lib.orc_mark(g.ctypes.data_as(_DP), C.byref(t), begin, end, tau_r, _p(vis), _p(q), _p(r))
        return vis, q, r

    def filter(self, tree, cam, tau_r, mode=2):
        t = orc_tree(tree)
        sel = np.zeros(max(1, tree.node_count()), np.uint32)
        n = C.c_uint64(0)
        ps, bs = C.c_int32(0), C.c_int32(0)
        c = cam.to_c()
        rc = self.lib.orc_filter(C.byref(t), C.byref(c), tau_r, mode, _p(sel), C.byref(n),
                                 C.byref(ps), C.byref(bs))
        if rc:
            raise L.ValidationError("oracle filter config")
        return sel[: n.value].copy(), ps.value, bs.value

    def effective_radius(self, sigma_max, opacity, kind, tau):
        err = C.c_int(0)
        r = self.lib.orc_effective_radius(sigma_max, opacity, kind, tau, C.byref(err))
        if err.value:
            raise L.ValidationError("shrink mode: tau in (0,1)")
        return r

    def prepare(self, tree, cam, selected, mode):
        sel = np.ascontiguousarray(selected, np.uint32)
        bl = L.BlendList.empty(max(1, sel.shape[0]))
        v = bl.view()
        t = orc_tree(tree)
        c = cam.to_c()
        rc = self.lib.orc_prepare(C.byref(t), C.byref(c), _p(sel), sel.shape[0], mode.kind,
                                  mode.tau, C.byref(v))
        if rc < 0:
            raise L.ValidationError("oracle prepare")
        return bl.truncated(rc)

    def bin_to_tiles(self, lst, w, h):
        v = lst.view()
        n = self.lib.orc_bin_count(C.byref(v), w, h)
        out = np.empty(n, L.PAIR_DTYPE)
        self.lib.orc_bin_to_tiles(C.byref(v), w, h, _p(out))
        return out

    def sort_pairs(self, pairs):
        self.lib.orc_sort_pairs(_p(pairs), pairs.shape[0])

    def exp_mx(self, x):
        return self.lib.orc_exp_mx(x)

    def alpha_blend(self, sorted_pairs, lst, w, h, kpc=False):
        img = np.zeros((h, w, 3), np.float32)
        k = np.zeros(sorted_pairs.shape[0], np.float64) if kpc else None
        v = lst.view()
        self.lib.orc_alpha_blend(_p(sorted_pairs), sorted_pairs.shape[0], C.byref(v), w, h,
                                 _p(img), _p(k))
        return (img, k) if kpc else img

    def render(self, tree, cam, tau_r, mode, collect_kpc=False):
        """Returns dict(image, selected, pairs, gaussians, stats, kpc)."""
        t = orc_tree(tree)
        c = cam.to_c()
        err = C.c_int(0)
        h = self.lib.orc_render(C.byref(t), C.byref(c), tau_r, mode.kind, mode.tau,
                                1 if collect_kpc else 0, C.byref(err))
        if not h:
            raise L.ValidationError(f"oracle render error {err.value}")
        try:
            st = OrcStats()
            self.lib.orc_render_stats(h, C.byref(st))
            W, H = cam.width, cam.height
            img = np.ctypeslib.as_array(C.cast(self.lib.orc_render_image(h), _FP),
                                        shape=(H * W * 3,)).reshape(H, W, 3).copy()
            sel = np.ctypeslib.as_array(C.cast(self.lib.orc_render_selected(h), C.POINTER(C.c_uint32)),
                                        shape=(max(1, st.n_selected),))[: st.n_selected].copy()
            np_ = st.n_pairs
            praw = C.cast(self.lib.orc_render_pairs(h), C.POINTER(C.c_uint8))
            pairs = np.frombuffer(C.string_at(praw, 12 * np_), dtype=L.PAIR_DTYPE).copy() if np_ else \
                np.empty(0, L.PAIR_DTYPE)
            kpc = None
            if collect_kpc and np_:
                kpc = np.ctypeslib.as_array(C.cast(self.lib.orc_render_kpc(h), _DP), shape=(np_,)).copy()
            v = L.BlendListC()
            self.lib.orc_render_gaussians(h, C.byref(v))
            ng = st.n_gaussians

            def arr(p, dt):
                if ng == 0:
                    return np.empty(0, dt)
                return np.ctypeslib.as_array(p, shape=(ng,)).copy()

            gl = L.BlendList(*[arr(getattr(v, f), np.float64) for f in L._LIST_F64],
                             depth=arr(v.depth, np.float32), node=arr(v.node, np.uint32))
            return dict(image=img, selected=sel, pairs=pairs, gaussians=gl, kpc=kpc,
                        n_selected=st.n_selected, n_pairs=np_, n_gaussians=ng,
                        passes=st.passes, barriers=st.barriers)
        finally:
            self.lib.orc_render_free(h)

    def psnr(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.orc_psnr(_p(a), _p(b), a.size)

    def view_gtc(self, pairs, kpc):
        return self.lib.orc_view_gtc(_p(pairs), _p(kpc), pairs.shape[0])


class Ref:
    """The reference library compiled in place (oracle/_ref)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_make_tree.restype = P
        lib.ref_make_tree.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_float, C.c_uint32,
                                      C.c_uint32, C.c_uint32]
        lib.ref_build_synthetic.restype = P
        lib.ref_build_synthetic.argtypes = [C.c_uint32, C.c_uint32, C.c_float, C.c_float, C.c_float,
                                            C.c_float, C.c_float, C.c_uint64, C.c_uint32, C.c_uint32,
                                            C.c_float, C.c_uint32, C.c_uint64]
        lib.ref_tree_from_arrays.restype = P
        lib.ref_tree_from_arrays.argtypes = [C.c_uint64, C.POINTER(_FP), P, P, P, C.c_uint32,
                                             C.c_float]
        lib.ref_tree_size.restype = C.c_uint64
        lib.ref_tree_size.argtypes = [P]
        lib.ref_tree_levels.restype = C.c_uint32
        lib.ref_tree_levels.argtypes = [P]
        lib.ref_tree_export.argtypes = [P, C.POINTER(_FP), P, P, P]
        lib.ref_tree_free.argtypes = [P]
        lib.ref_validate_tree.restype = C.c_uint64
        lib.ref_validate_tree.argtypes = [P]
        lib.ref_rng_new.restype = P
        lib.ref_rng_new.argtypes = [C.c_uint64]
        lib.ref_rng_free.argtypes = [P]
        lib.ref_rng_next_u64.restype = C.c_uint64
        lib.ref_rng_next_u64.argtypes = [P]
        lib.ref_rng_uniform.restype = C.c_double
        lib.ref_rng_uniform.argtypes = [P, C.c_double, C.c_double]
        lib.ref_rng_next_below.restype = C.c_uint64
        lib.ref_rng_next_below.argtypes = [P, C.c_uint64]
        lib.ref_mix_seed.restype = C.c_uint64
        lib.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.ref_orbit_camera.argtypes = [P, C.c_uint32, C.c_uint32, C.c_double, C.POINTER(CameraC)]
        lib.ref_front_camera.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.POINTER(CameraC)]
        lib.ref_camera_path_sample.argtypes = [C.POINTER(CameraC), C.c_uint32, P, C.POINTER(CameraC)]
        lib.ref_camera_geom.argtypes = [C.POINTER(CameraC), _DP]
        lib.ref_mark.argtypes = [P, C.POINTER(CameraC), C.c_uint64, C.c_uint64, C.c_double, P, P, P,
                                 C.c_int]
        lib.ref_exp_mx.restype = C.c_double
        lib.ref_exp_mx.argtypes = [C.c_double]
        lib.ref_effective_radius.restype = C.c_double
        lib.ref_effective_radius.argtypes = [C.c_double, C.c_float, C.c_int, C.c_double]
        lib.ref_filter.argtypes = [P, C.POINTER(CameraC), C.c_double, C.c_uint32, C.c_int, P,
                                   C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int32), _DP, _DP]
        lib.ref_prepare.argtypes = [P, C.POINTER(CameraC), P, C.c_uint64, C.c_int, C.c_double,
                                    C.POINTER(L.BlendListC)]
        lib.ref_bin_to_tiles.restype = P
        lib.ref_bin_to_tiles.argtypes = [C.POINTER(L.BlendListC), C.c_int, C.c_int,
                                         C.POINTER(C.c_uint64)]
        lib.ref_pairs_copy.argtypes = [P, P]
        lib.ref_pairs_free.argtypes = [P]
        lib.ref_sort_pairs.argtypes = [P, C.c_uint64]
        lib.ref_alpha_blend.argtypes = [P, C.c_uint64, C.POINTER(L.BlendListC), C.c_int, C.c_int,
                                        C.c_uint32, P, P]
        lib.ref_render.restype = P
        lib.ref_render.argtypes = [P, C.POINTER(CameraC), C.c_double, C.c_int, C.c_double,
                                   C.c_uint32, C.c_int, C.c_int, C.POINTER(RefStats)]
        lib.ref_render_image.argtypes = [P, P]
        lib.ref_render_pairs.argtypes = [P, P, P]
        lib.ref_render_gaussians.argtypes = [P, C.POINTER(L.BlendListC)]
        lib.ref_render_free.argtypes = [P]
        lib.ref_calibrate.argtypes = [P, C.POINTER(CameraC), C.c_uint32, C.c_double, C.c_double,
                                      C.c_uint32, _DP, _DP, _DP, C.POINTER(C.c_uint32), P]
        lib.ref_view_gtc.restype = C.c_double
        lib.ref_view_gtc.argtypes = [P, P, C.c_uint64]
        lib.ref_psnr.restype = C.c_double
        lib.ref_psnr.argtypes = [P, P, C.c_int, C.c_int]
        lib.ref_ssim.restype = C.c_double
        lib.ref_ssim.argtypes = [P, P, C.c_int, C.c_int]
        self.lib = lib

    def err(self):
        return self.lib.ref_last_error().decode()

    # --- trees ---
    def export(self, h, shrink=0.5) -> L.LoDTree:
        n = self.lib.ref_tree_size(h)
        nl = self.lib.ref_tree_levels(h)
        t = L.LoDTree.empty(n, nl, shrink)
        ptrs = (_FP * 14)(*[getattr(t, f).ctypes.data_as(_FP) for f in L._FIELDS])
        self.lib.ref_tree_export(h, ptrs, _p(t.parent), _p(t.leaf), _p(t.level_offsets))
        return t

    def make_tree(self, seed, depth, children=8, gamma=0.5, nx=3, ny=3, congestion=1):
        """Returns (handle, exported LoDTree)."""
        h = self.lib.ref_make_tree(seed, depth, children, gamma, nx, ny, congestion)
        if not h:
            raise L.ValidationError(self.err())
        return h, self.export(h, gamma)

    def build_synthetic(self, nx, ny, spacing=2.0, scale_min=0.2, scale_max=0.6, opacity_min=0.3,
                        opacity_max=0.9, seed=0, congestion=1, depth=3, shrink=0.5, children=8,
                        build_seed=0):
        h = self.lib.ref_build_synthetic(nx, ny, spacing, scale_min, scale_max, opacity_min,
                                         opacity_max, seed, congestion, depth, shrink, children,
                                         build_seed)
        if not h:
            raise L.ValidationError(self.err())
        return h, self.export(h, shrink)

    def tree_from(self, t: L.LoDTree):
        ptrs = (_FP * 14)(*[getattr(t, f).ctypes.data_as(_FP) for f in L._FIELDS])
        return self.lib.ref_tree_from_arrays(t.node_count(), ptrs, _p(t.parent), _p(t.leaf),
                                             _p(t.level_offsets), t.level_count(),
                                             float(t.shrink_factor))

    def free_tree(self, h):
        self.lib.ref_tree_free(h)

    def validate(self, h):
        return self.lib.ref_validate_tree(h)

    # --- rng / cameras ---
    def rng(self, seed):
        return self.lib.ref_rng_new(seed)

    def orbit_camera(self, rng, w, h, dist):
        c = CameraC()
        self.lib.ref_orbit_camera(rng, w, h, dist, C.byref(c))
        return L.Camera.from_c(c)

    def front_camera(self, w, h, focal=100.0):
        c = CameraC()
        self.lib.ref_front_camera(w, h, focal, C.byref(c))
        return L.Camera.from_c(c)

    def camera_geom(self, cam):
        out = np.zeros(44)
        c = cam.to_c()
        self.lib.ref_camera_geom(C.byref(c), out.ctypes.data_as(_DP))
        return out

    def sample_path(self, keys, samples):
        n = sum(samples) + 1
        kc = (CameraC * len(keys))(*[k.to_c() for k in keys])
        s = np.asarray(samples, np.uint32)
        out = (CameraC * n)()
        rc = self.lib.ref_camera_path_sample(kc, len(keys), _p(s), out)
        if rc:
            raise L.ValidationError(self.err())
        return [L.Camera.from_c(out[i]) for i in range(n)]

    # --- path ---
    def mark(self, h, n, cam, tau_r, begin=0, end=None, backend=0):
        end = n if end is None else end
        vis = np.full(n, 7, np.uint8)
        q = np.full(n, 7, np.uint8)
        r = np.full(n, -1.0)
        c = cam.to_c()
        rc = self.lib.ref_mark(h, C.byref(c), begin, end, tau_r, _p(vis), _p(q), _p(r), backend)
        assert rc == 0, self.err()
        return vis, q, r

    def filter(self, h, n, cam, tau_r, mode=2, workers=1):
        sel = np.zeros(max(1, n), np.uint32)
        k = C.c_uint64(0)
        ps, bs = C.c_int32(0), C.c_int32(0)
        c = cam.to_c()
        rc = self.lib.ref_filter(h, C.byref(c), tau_r, workers, mode, _p(sel), max(1, n), C.byref(k),
                                 C.byref(ps), C.byref(bs), None, None)
        if rc:
            raise L.ValidationError(self.err())
        return sel[: k.value].copy(), ps.value, bs.value

    def prepare(self, h, cam, selected, mode):
        sel = np.ascontiguousarray(selected, np.uint32)
        bl = L.BlendList.empty(max(1, sel.shape[0]))
        v = bl.view()
        c = cam.to_c()
        rc = self.lib.ref_prepare(h, C.byref(c), _p(sel), sel.shape[0], mode.kind, mode.tau, C.byref(v))
        if rc:
            raise L.ValidationError(self.err())
        return bl.truncated(int(v.n))

    def bin_to_tiles(self, lst, w, h):
        v = lst.view()
        n = C.c_uint64(0)
        hp = self.lib.ref_bin_to_tiles(C.byref(v), w, h, C.byref(n))
        out = np.empty(n.value, L.PAIR_DTYPE)
        self.lib.ref_pairs_copy(hp, _p(out))
        self.lib.ref_pairs_free(hp)
        return out

    def sort_pairs(self, pairs):
        self.lib.ref_sort_pairs(_p(pairs), pairs.shape[0])

    def alpha_blend(self, sorted_pairs, lst, w, h, workers=1, kpc=False):
        img = np.zeros((h, w, 3), np.float32)
        k = np.zeros(sorted_pairs.shape[0]) if kpc else None
        v = lst.view()
        rc = self.lib.ref_alpha_blend(_p(sorted_pairs), sorted_pairs.shape[0], C.byref(v), w, h,
                                      workers, _p(img), _p(k))
        assert rc == 0, self.err()
        return (img, k) if kpc else img

    def exp_mx(self, x):
        return self.lib.ref_exp_mx(x)

    def effective_radius(self, sigma_max, opacity, kind, tau):
        return self.lib.ref_effective_radius(sigma_max, opacity, kind, tau)

    def render(self, h, cam, tau_r, mode, workers=1, collect_kpc=False, filter_mode=0):
        st = RefStats()
        c = cam.to_c()
        r = self.lib.ref_render(h, C.byref(c), tau_r, mode.kind, mode.tau, workers, filter_mode,
                                1 if collect_kpc else 0, C.byref(st))
        if not r:
            raise L.ValidationError(self.err())
        try:
            img = np.zeros((cam.height, cam.width, 3), np.float32)
            self.lib.ref_render_image(r, _p(img))
            out = dict(image=img, n_selected=st.n_selected, n_pairs=st.n_pairs,
                       passes=st.passes, barriers=st.barriers,
                       total_ms=st.t_calc_ms + st.t_sync_ms + st.t_prepr_ms + st.t_sort_ms + st.t_alpha_ms,
                       stage_ms=(st.t_calc_ms, st.t_sync_ms, st.t_prepr_ms, st.t_sort_ms, st.t_alpha_ms))
            if collect_kpc:
                pairs = np.empty(st.n_pairs, L.PAIR_DTYPE)
                kpc = np.empty(st.n_pairs)
                self.lib.ref_render_pairs(r, _p(pairs), _p(kpc))
                bl = L.BlendList.empty(max(1, st.n_gaussians))
                v = bl.view()
                self.lib.ref_render_gaussians(r, C.byref(v))
                out.update(pairs=pairs, kpc=kpc, gaussians=bl.truncated(st.n_gaussians),
                           n_gaussians=st.n_gaussians)
            return out
        finally:
            self.lib.ref_render_free(r)

    def psnr(self, a, b):
        h, w = a.shape[:2]
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.ref_psnr(_p(a), _p(b), w, h)

    def ssim(self, a, b):
        h, w = a.shape[:2]
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.ref_ssim(_p(a), _p(b), w, h)

