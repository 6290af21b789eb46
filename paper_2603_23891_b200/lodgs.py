"""Python mirror of the reference ``lodgs`` per-frame render API, on the B200 kernels.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/lodgs/{scene,filter,rasterizer}.hpp):

* ``LoDTree`` (scene.hpp:29-74), ``Camera`` (scene.hpp:76-82),
  ``FilterConfig`` / ``FilterResult`` (filter.hpp:11-22),
  ``ShrinkMode`` (rasterizer.hpp:16-24), ``RenderOptions`` / ``RenderStats`` /
  ``RenderOutput`` (rasterizer.hpp:73-104), ``BlendList`` (rasterizer.hpp:36-51),
  ``TileGrid`` / tile pairs (tiles.hpp:11-34).
* ``render`` (rasterizer.hpp:106-108), ``filter_parallel`` (filter.hpp:42-43),
  ``prepare_gaussians`` / ``bin_to_tiles`` / ``sort_pairs`` / ``alpha_blend``
  (rasterizer.hpp:55-71).
* ``ValidationError`` / ``IoError`` / ``FormatError`` (core.hpp:91-103).

Every compute call goes through the C ABI in ``include/lodgs_gpu.h``
(``_lib/liblodgs_b200.so``) onto hand-written sm_100a kernels.  There is no
CPU fallback: without the library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "liblodgs_b200.so")
# experiment builds (tools/variants.sh) may point elsewhere; the product default is _lib/
LIB_PATH = os.environ.get("LODGS_B200_LIB", LIB_PATH)

ROOT_PARENT = 0xFFFFFFFF  # core.hpp:15
_BLEND_FLAGS = {"cpa": 0, "wsp": 512, "tma": 64, "gather4": 128}  # LODGS_RENDER_BLEND_*
TILE = 16  # tiles.hpp:8-9

# --------------------------------------------------------------- errors --


class ValidationError(RuntimeError):
    """core.hpp:91-93 -- contract violations (status 2)."""


class FormatError(ValidationError):
    """core.hpp:101-103 -- malformed content (status 2)."""


class IoError(RuntimeError):
    """core.hpp:96-98 -- filesystem failures (status 3)."""


class CudaError(RuntimeError):
    """CUDA runtime failure or no usable device (status 4)."""


class InternalError(RuntimeError):
    """Internal error, e.g. pair-buffer overflow reported by render_async (status 5)."""


# ------------------------------------------------------------- ctypes ABI --


class CameraC(C.Structure):
    _fields_ = [
        ("width", C.c_uint32),
        ("height", C.c_uint32),
        ("fx", C.c_double),
        ("fy", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("rotation", C.c_double * 9),
        ("translation", C.c_double * 3),
        ("znear", C.c_double),
        ("zfar", C.c_double),
    ]


_FP = C.POINTER(C.c_float)


class TreeViewC(C.Structure):
    _fields_ = [("n_nodes", C.c_uint64)] + [
        (name, _FP)
        for name in (
            "mean_x", "mean_y", "mean_z", "scale_x", "scale_y", "scale_z",
            "quat_w", "quat_x", "quat_y", "quat_z", "opacity",
            "color_r", "color_g", "color_b",
        )
    ] + [
        ("parent", C.POINTER(C.c_uint32)),
        ("leaf", C.POINTER(C.c_uint8)),
        ("level_offsets", C.POINTER(C.c_uint32)),
        ("n_levels", C.c_uint32),
        ("shrink_factor", C.c_float),
    ]


class TreeBuffersC(C.Structure):
    _fields_ = [
        (name, _FP)
        for name in (
            "mean_x", "mean_y", "mean_z", "scale_x", "scale_y", "scale_z",
            "quat_w", "quat_x", "quat_y", "quat_z", "opacity",
            "color_r", "color_g", "color_b",
        )
    ] + [
        ("parent", C.POINTER(C.c_uint32)),
        ("leaf", C.POINTER(C.c_uint8)),
        ("level_offsets", C.POINTER(C.c_uint32)),
    ]


class SyntheticSpecC(C.Structure):
    _fields_ = [
        ("nx", C.c_uint32), ("ny", C.c_uint32), ("spacing", C.c_float),
        ("scale_min", C.c_float), ("scale_max", C.c_float),
        ("opacity_min", C.c_float), ("opacity_max", C.c_float),
        ("seed", C.c_uint64), ("congestion", C.c_uint32),
    ]


class BuildConfigC(C.Structure):
    _fields_ = [
        ("depth", C.c_uint32), ("shrink_factor", C.c_float),
        ("children_per_node", C.c_uint32), ("seed", C.c_uint64),
    ]


class RenderParamsC(C.Structure):
    _fields_ = [
        ("tau_r", C.c_double), ("tau", C.c_double),
        ("shrink_kind", C.c_int32), ("flags", C.c_uint32),
    ]


class RenderStatsC(C.Structure):
    _fields_ = [
        ("n_selected", C.c_uint64), ("n_gaussians", C.c_uint64), ("n_pairs", C.c_uint64),
        ("filter_passes", C.c_int32), ("filter_barriers", C.c_int32),
        ("t_calc_ms", C.c_double), ("t_sync_ms", C.c_double), ("t_prepr_ms", C.c_double),
        ("t_sort_ms", C.c_double), ("t_alpha_ms", C.c_double),
        ("big_tiles", C.c_uint32), ("kernel_launches", C.c_uint32),
    ]


_DP = C.POINTER(C.c_double)


class BlendListC(C.Structure):
    _fields_ = [("n", C.c_uint64)] + [
        (name, _DP)
        for name in ("mean_x", "mean_y", "conic_a", "conic_b", "conic_c", "opacity",
                     "col_r", "col_g", "col_b", "radius")
    ] + [("depth", _FP), ("node", C.POINTER(C.c_uint32))]


class CalibrationC(C.Structure):
    _fields_ = [("tau", C.c_double), ("scene_gtc", C.c_double), ("lambda_g", C.c_double),
                ("n_views", C.c_uint32), ("histogram", C.c_uint64 * 5)]


PAIR_DTYPE = np.dtype([("tile", "<u4"), ("depth", "<f4"), ("gaussian", "<u4")])

# C ABI symbols declared by include/lodgs_gpu.h (checked by tests).
ABI_SYMBOLS = (
    "lodgs_gpu_last_error", "lodgs_gpu_abi_version", "lodgs_gpu_device_count",
    "lodgs_validate_tree", "lodgs_validate_camera", "lodgs_camera_geom",
    "lodgs_gpu_scene_create", "lodgs_gpu_scene_destroy", "lodgs_gpu_scene_stream",
    "lodgs_gpu_scene_reserve", "lodgs_gpu_scene_memory", "lodgs_gpu_render",
    "lodgs_gpu_render_batch",
    "lodgs_gpu_render_async", "lodgs_gpu_sync", "lodgs_gpu_take_totals",
    "lodgs_gpu_profile", "lodgs_gpu_profile_read",
    "lodgs_gpu_read_image", "lodgs_gpu_image_device_ptr", "lodgs_gpu_read_selected",
    "lodgs_gpu_read_pairs", "lodgs_gpu_read_gaussians", "lodgs_gpu_read_counts",
    "lodgs_gpu_read_kpc", "lodgs_gpu_calibrate",
    "lodgs_gpu_filter", "lodgs_gpu_filter_serial", "lodgs_gpu_mark", "lodgs_gpu_prepare", "lodgs_gpu_bin_to_tiles",
    "lodgs_gpu_sort_pairs", "lodgs_gpu_alpha_blend", "lodgs_gpu_host_alloc",
    "lodgs_gpu_host_free", "lodgs_gpu_read_image_rgb8", "lodgs_gpu_set_reference_image",
    "lodgs_gpu_compare_reference", "lodgs_gpu_image_metrics", "lodgs_gpu_scene_load",
    "lodgs_gpu_scene_info", "lodgs_gpu_scene_set_inflight", "lodgs_gpu_join",
    "lodgs_gpu_scene_set_sh", "lodgs_gpu_render_views_async",
)

_lib = None


def load_library():
    """Loads _lib/liblodgs_b200.so (built by __graft_entry__.build()). Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback."
        )
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sig = {
        "lodgs_gpu_last_error": (C.c_char_p, []),
        "lodgs_gpu_abi_version": (C.c_int, []),
        "lodgs_gpu_device_count": (C.c_int, [C.POINTER(C.c_int)]),
        "lodgs_validate_tree": (C.c_int, [C.POINTER(TreeViewC), C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]),
        "lodgs_validate_camera": (C.c_int, [C.POINTER(CameraC), C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]),
        "lodgs_camera_geom": (C.c_int, [C.POINTER(CameraC), _DP]),
        "lodgs_gpu_scene_create": (C.c_int, [C.POINTER(TreeViewC), C.c_int, C.POINTER(P)]),
        "lodgs_gpu_scene_destroy": (C.c_int, [P]),
        "lodgs_gpu_scene_stream": (C.c_int, [P, C.POINTER(P)]),
        "lodgs_gpu_scene_reserve": (C.c_int, [P, C.c_uint64]),
        "lodgs_gpu_scene_memory": (C.c_int, [P, C.POINTER(C.c_uint64)]),
        "lodgs_gpu_render": (C.c_int, [P, C.POINTER(CameraC), C.POINTER(RenderParamsC), P,
                                       C.POINTER(RenderStatsC)]),
        "lodgs_gpu_render_batch": (C.c_int, [P, C.POINTER(CameraC), C.c_uint64,
                                             C.POINTER(RenderParamsC), C.POINTER(P),
                                             C.POINTER(RenderStatsC)]),
        "lodgs_gpu_render_async": (C.c_int, [P, C.POINTER(CameraC), C.POINTER(RenderParamsC), P]),
        "lodgs_gpu_sync": (C.c_int, [P, C.POINTER(RenderStatsC)]),
        "lodgs_gpu_take_totals": (C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                             C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "lodgs_gpu_profile": (C.c_int, [P, C.c_int]),
        "lodgs_gpu_profile_read": (C.c_int, [P, C.POINTER(C.c_uint64), _DP]),
        "lodgs_gpu_read_image": (C.c_int, [P, P]),
        "lodgs_gpu_image_device_ptr": (C.c_int, [P, C.POINTER(P)]),
        "lodgs_gpu_read_selected": (C.c_int, [P, P, C.c_uint64, C.POINTER(C.c_uint64)]),
        "lodgs_gpu_read_pairs": (C.c_int, [P, P, C.c_uint64, C.POINTER(C.c_uint64)]),
        "lodgs_gpu_read_gaussians": (C.c_int, [P, C.POINTER(BlendListC), C.c_uint64]),
        "lodgs_gpu_read_counts": (C.c_int, [P, P, C.c_uint64, P, C.c_uint64]),
        "lodgs_gpu_read_kpc": (C.c_int, [P, P, C.c_uint64, C.POINTER(C.c_uint64)]),
        "lodgs_gpu_calibrate": (C.c_int, [P, C.POINTER(CameraC), C.c_uint32, C.c_double,
                                          C.c_double, C.POINTER(CalibrationC), _DP]),
        "lodgs_gpu_filter": (C.c_int, [P, C.POINTER(CameraC), C.c_double, P, C.c_uint64,
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32)]),
        "lodgs_gpu_read_image_rgb8": (C.c_int, [P, P]),
        "lodgs_gpu_scene_set_inflight": (C.c_int, [P, C.c_int]),
        "lodgs_gpu_scene_set_sh": (C.c_int, [P, C.c_int, P, C.c_uint64]),
        "lodgs_gpu_render_views_async": (C.c_int, [P, P, C.c_uint64, P, P]),
        "lodgs_gpu_join": (C.c_int, [P]),
        "lodgs_gpu_scene_load": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(P), _DP]),
        "lodgs_gpu_scene_info": (C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), P,
                                           C.c_uint32, C.POINTER(C.c_float)]),
        "lodgs_gpu_set_reference_image": (C.c_int, [P]),
        "lodgs_gpu_compare_reference": (C.c_int, [P, _DP, _DP]),
        "lodgs_gpu_image_metrics": (C.c_int, [P, P, C.c_int, C.c_int, _DP, _DP]),
        "lodgs_gpu_filter_serial": (C.c_int, [P, C.POINTER(CameraC), C.c_double, P, C.c_uint64,
                                              C.POINTER(C.c_uint64), C.POINTER(C.c_int32),
                                              C.POINTER(C.c_int32), _DP]),
        "lodgs_gpu_mark": (C.c_int, [P, C.POINTER(CameraC), C.c_uint64, C.c_uint64, C.c_double,
                                     P, P, P]),
        "lodgs_gpu_prepare": (C.c_int, [P, C.POINTER(CameraC), P, C.c_uint64, C.c_int32,
                                        C.c_double, C.POINTER(BlendListC)]),
        "lodgs_gpu_bin_to_tiles": (C.c_int, [C.POINTER(BlendListC), C.c_int, C.c_int, P,
                                             C.c_uint64, C.POINTER(C.c_uint64)]),
        "lodgs_gpu_sort_pairs": (C.c_int, [P, C.c_uint64]),
        "lodgs_gpu_alpha_blend": (C.c_int, [P, C.c_uint64, C.POINTER(BlendListC), C.c_int,
                                            C.c_int, C.c_uint32, P]),
        "lodgs_gpu_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(P)]),
        "lodgs_gpu_host_free": (C.c_int, [P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


SYNTH_PATH = os.path.join(_HERE, "_lib", "liblodgs_synth.so")
SYNTH_SYMBOLS = ("lodgs_synth_last_error", "lodgs_camera_path_sample", "lodgs_build_synthetic_tree")
_synth = None


def load_synth_library():
    """_lib/liblodgs_synth.so (include/lodgs_synth.h): benchmark INPUT generation -- the
    reference's synthetic tree generator and CameraPath::sample restated -- kept out of
    the renderer library."""
    global _synth
    if _synth is not None:
        return _synth
    if not os.path.exists(SYNTH_PATH):
        raise ImportError(f"{SYNTH_PATH} is missing: run __graft_entry__.build()")
    lib = C.CDLL(SYNTH_PATH)
    lib.lodgs_synth_last_error.restype = C.c_char_p
    lib.lodgs_synth_last_error.argtypes = []
    lib.lodgs_camera_path_sample.restype = C.c_int
    lib.lodgs_camera_path_sample.argtypes = [C.POINTER(CameraC), C.c_uint32, C.POINTER(C.c_uint32),
                                             C.POINTER(CameraC), C.c_uint64, C.POINTER(C.c_uint64)]
    lib.lodgs_build_synthetic_tree.restype = C.c_int
    lib.lodgs_build_synthetic_tree.argtypes = [C.POINTER(SyntheticSpecC), C.POINTER(BuildConfigC),
                                               C.POINTER(TreeBuffersC), C.POINTER(C.c_uint64),
                                               C.POINTER(C.c_uint32)]
    _synth = lib
    return lib


def _check_synth(rc: int):
    if rc == 0:
        return
    msg = load_synth_library().lodgs_synth_last_error().decode(errors="replace")
    raise (ValidationError if rc == 2 else InternalError)(msg)


def _check(rc: int):
    if rc == 0:
        return
    msg = load_library().lodgs_gpu_last_error().decode(errors="replace")
    if rc == 2:
        raise ValidationError(msg)
    if rc == 3:
        raise IoError(msg)
    if rc == 4:
        raise CudaError(msg)
    raise InternalError(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def device_count() -> int:
    n = C.c_int(0)
    rc = load_library().lodgs_gpu_device_count(C.byref(n))
    return n.value if rc == 0 else 0


# ------------------------------------------------------------ data model --

_FIELDS = ("mean_x", "mean_y", "mean_z", "scale_x", "scale_y", "scale_z",
           "quat_w", "quat_x", "quat_y", "quat_z", "opacity", "color_r", "color_g", "color_b")


@dataclasses.dataclass
class Camera:
    """scene.hpp:76-82 -- pinhole camera, world->camera rotation (row-major) + translation."""

    width: int = 0
    height: int = 0
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    rotation: Sequence[float] = (1, 0, 0, 0, 1, 0, 0, 0, 1)
    translation: Sequence[float] = (0, 0, 0)
    near: float = 0.01
    far: float = 1000.0

    def to_c(self) -> CameraC:
        c = CameraC()
        c.width, c.height = int(self.width), int(self.height)
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        for i in range(9):
            c.rotation[i] = float(self.rotation[i])
        for i in range(3):
            c.translation[i] = float(self.translation[i])
        c.znear, c.zfar = float(self.near), float(self.far)
        return c

    @staticmethod
    def from_c(c: CameraC) -> "Camera":
        return Camera(c.width, c.height, c.fx, c.fy, c.cx, c.cy, tuple(c.rotation),
                      tuple(c.translation), c.znear, c.zfar)


@dataclasses.dataclass
class LoDTree:
    """scene.hpp:29-74 -- level-major SoA node arena (numpy arrays)."""

    mean_x: np.ndarray
    mean_y: np.ndarray
    mean_z: np.ndarray
    scale_x: np.ndarray
    scale_y: np.ndarray
    scale_z: np.ndarray
    quat_w: np.ndarray
    quat_x: np.ndarray
    quat_y: np.ndarray
    quat_z: np.ndarray
    opacity: np.ndarray
    color_r: np.ndarray
    color_g: np.ndarray
    color_b: np.ndarray
    parent: np.ndarray
    leaf: np.ndarray
    level_offsets: np.ndarray
    shrink_factor: float = 0.5

    def __post_init__(self):
        for f in _FIELDS:
            setattr(self, f, np.ascontiguousarray(getattr(self, f), dtype=np.float32))
        self.parent = np.ascontiguousarray(self.parent, dtype=np.uint32)
        self.leaf = np.ascontiguousarray(self.leaf, dtype=np.uint8)
        self.level_offsets = np.ascontiguousarray(self.level_offsets, dtype=np.uint32)

    def node_count(self) -> int:
        return int(self.mean_x.shape[0])

    def level_count(self) -> int:
        return int(self.level_offsets.shape[0])

    def level_begin(self, l: int) -> int:
        return int(self.level_offsets[l])

    def level_end(self, l: int) -> int:
        return int(self.level_offsets[l + 1]) if l + 1 < self.level_count() else self.node_count()

    def view(self) -> TreeViewC:
        v = TreeViewC()
        v.n_nodes = self.node_count()
        for f in _FIELDS:
            setattr(v, f, getattr(self, f).ctypes.data_as(_FP))
        v.parent = self.parent.ctypes.data_as(C.POINTER(C.c_uint32))
        v.leaf = self.leaf.ctypes.data_as(C.POINTER(C.c_uint8))
        v.level_offsets = self.level_offsets.ctypes.data_as(C.POINTER(C.c_uint32))
        v.n_levels = self.level_count()
        v.shrink_factor = float(self.shrink_factor)
        return v

    @staticmethod
    def empty(n: int, n_levels: int, shrink_factor: float = 0.5) -> "LoDTree":
        z = {f: np.zeros(n, np.float32) for f in _FIELDS}
        return LoDTree(**z, parent=np.zeros(n, np.uint32), leaf=np.zeros(n, np.uint8),
                       level_offsets=np.zeros(n_levels, np.uint32), shrink_factor=shrink_factor)


@dataclasses.dataclass
class FilterConfig:
    """filter.hpp:11-14.  worker_count is accepted for API parity; the GPU ignores it."""

    tau_r: float = 3.0
    worker_count: int = 1


@dataclasses.dataclass
class FilterResult:
    """filter.hpp:16-22."""

    selected: np.ndarray
    passes: int = 0
    barriers: int = 0
    calc_ms: float = 0.0
    sync_ms: float = 0.0


@dataclasses.dataclass
class ShrinkMode:
    """rasterizer.hpp:16-24."""

    kind: int = 0  # 0 three_sigma, 1 fixed, 2 adaptive
    tau: float = 0.0
    THREE_SIGMA = 0
    FIXED = 1
    ADAPTIVE = 2

    @staticmethod
    def three_sigma() -> "ShrinkMode":
        return ShrinkMode(0, 0.0)

    @staticmethod
    def fixed() -> "ShrinkMode":
        return ShrinkMode(1, 1.0 / 255.0)

    @staticmethod
    def adaptive(tau: float) -> "ShrinkMode":
        return ShrinkMode(2, float(tau))


@dataclasses.dataclass
class RenderOptions:
    """rasterizer.hpp:100-104, plus B200 switches (exact_blend, stage_timing)."""

    worker_count: int = 1
    collect_kpc: bool = False
    filter_mode: str = "parallel"
    exact_blend: bool = False
    stage_timing: bool = False
    output_rgb8: bool = False  # render_batch host images are W*H*3 bytes (save_ppm quantisation)
    # fast-blend kernel: "wsp" (default, cp.async producer warps), "tma" (sort-written
    # records streamed with cp.async.bulk), "gather4" (TMA tile::gather4); DESIGN.md 3.7
    blend_kernel: str = "cpa"


@dataclasses.dataclass
class RenderStats:
    """rasterizer.hpp:73-84."""

    n_selected: int = 0
    n_pairs: int = 0
    n_gaussians: int = 0
    filter_passes: int = 0
    filter_barriers: int = 0
    t_calc_ms: float = 0.0
    t_sync_ms: float = 0.0
    t_prepr_ms: float = 0.0
    t_sort_ms: float = 0.0
    t_alpha_ms: float = 0.0
    big_tiles: int = 0
    kernel_launches: int = 0  # sm_100a kernels enqueued for the frame

    def total_ms(self) -> float:
        return self.t_calc_ms + self.t_sync_ms + self.t_prepr_ms + self.t_sort_ms + self.t_alpha_ms

    @staticmethod
    def from_c(s: RenderStatsC) -> "RenderStats":
        return RenderStats(s.n_selected, s.n_pairs, s.n_gaussians, s.filter_passes,
                           s.filter_barriers, s.t_calc_ms, s.t_sync_ms, s.t_prepr_ms,
                           s.t_sort_ms, s.t_alpha_ms, s.big_tiles, s.kernel_launches)


_LIST_F64 = ("mean_x", "mean_y", "conic_a", "conic_b", "conic_c", "opacity",
             "col_r", "col_g", "col_b", "radius")


@dataclasses.dataclass
class BlendList:
    """rasterizer.hpp:36-51 -- compacted screen-space gaussians (FP64)."""

    mean_x: np.ndarray
    mean_y: np.ndarray
    conic_a: np.ndarray
    conic_b: np.ndarray
    conic_c: np.ndarray
    opacity: np.ndarray
    col_r: np.ndarray
    col_g: np.ndarray
    col_b: np.ndarray
    radius: np.ndarray
    depth: np.ndarray
    node: np.ndarray

    def __post_init__(self):
        for f in _LIST_F64:
            setattr(self, f, np.ascontiguousarray(getattr(self, f), dtype=np.float64))
        self.depth = np.ascontiguousarray(self.depth, dtype=np.float32)
        self.node = np.ascontiguousarray(self.node, dtype=np.uint32)

    def size(self) -> int:
        return int(self.mean_x.shape[0])

    @staticmethod
    def empty(n: int) -> "BlendList":
        return BlendList(*[np.zeros(n, np.float64) for _ in _LIST_F64],
                         depth=np.zeros(n, np.float32), node=np.zeros(n, np.uint32))

    def view(self) -> BlendListC:
        v = BlendListC()
        v.n = self.size()
        for f in _LIST_F64:
            setattr(v, f, getattr(self, f).ctypes.data_as(_DP))
        v.depth = self.depth.ctypes.data_as(_FP)
        v.node = self.node.ctypes.data_as(C.POINTER(C.c_uint32))
        return v

    def truncated(self, n: int) -> "BlendList":
        return BlendList(*[getattr(self, f)[:n].copy() for f in _LIST_F64],
                         depth=self.depth[:n].copy(), node=self.node[:n].copy())


@dataclasses.dataclass
class TileGrid:
    """tiles.hpp:11-21."""

    tiles_x: int
    tiles_y: int

    @staticmethod
    def make(width: int, height: int) -> "TileGrid":
        return TileGrid((width + TILE - 1) // TILE, (height + TILE - 1) // TILE)

    def n_tile(self) -> int:
        return self.tiles_x * self.tiles_y

    def tile_id(self, tx: int, ty: int) -> int:
        return ty * self.tiles_x + tx


@dataclasses.dataclass
class Image:
    """image.hpp:10-23 -- interleaved RGB f32, shape (H, W, 3)."""

    width: int
    height: int
    rgb: np.ndarray


@dataclasses.dataclass
class CalibrationReport:
    """metrics.hpp:44-54."""

    per_view: np.ndarray
    scene_mean: float
    lambda_g: float
    tau: float
    n_views: int
    histogram: list


@dataclasses.dataclass
class RenderOutput:
    """rasterizer.hpp:86-96."""

    image: Image
    stats: RenderStats
    pairs: Optional[np.ndarray] = None
    kpc: Optional[np.ndarray] = None
    gaussians: Optional[BlendList] = None


# ------------------------------------------------------- host utilities --


def validate_tree(tree: LoDTree) -> int:
    """scene.cpp:89-165 -- number of rule violations."""
    n = C.c_uint64(0)
    v = tree.view()
    _check(load_library().lodgs_validate_tree(C.byref(v), C.byref(n), None, 0))
    return int(n.value)


def require_valid(tree: LoDTree) -> None:
    n = C.c_uint64(0)
    buf = C.create_string_buffer(4096)
    v = tree.view()
    _check(load_library().lodgs_validate_tree(C.byref(v), C.byref(n), buf, 4096))
    if n.value:
        raise ValidationError(buf.value.decode())


def camera_geom(cam: Camera) -> np.ndarray:
    """projection.cpp:11-38 CameraGeom::make -> 44 doubles."""
    out = np.zeros(44, np.float64)
    c = cam.to_c()
    _check(load_library().lodgs_camera_geom(C.byref(c), out.ctypes.data_as(_DP)))
    return out


def sample_camera_path(keyframes: Sequence[Camera], samples: Sequence[int]) -> list:
    """camera_path.cpp:132-142 CameraPath::sample."""
    lib = load_synth_library()
    keys = (CameraC * len(keyframes))(*[k.to_c() for k in keyframes])
    smp = (C.c_uint32 * max(1, len(samples)))(*samples)
    n = C.c_uint64(0)
    _check_synth(lib.lodgs_camera_path_sample(keys, len(keyframes), smp, None, 0, C.byref(n)))
    out = (CameraC * n.value)()
    _check_synth(lib.lodgs_camera_path_sample(keys, len(keyframes), smp, out, n.value, C.byref(n)))
    return [Camera.from_c(out[i]) for i in range(n.value)]


def build_synthetic_tree(nx=8, ny=8, spacing=2.0, scale_min=0.2, scale_max=0.6,
                         opacity_min=0.3, opacity_max=0.9, seed=0, congestion=1,
                         depth=3, shrink_factor=0.5, children_per_node=8,
                         build_seed=0) -> LoDTree:
    """build_tree(generate_synthetic_scene(spec), cfg) -- tree_builder.cpp:75-174."""
    lib = load_synth_library()
    spec = SyntheticSpecC(nx, ny, spacing, scale_min, scale_max, opacity_min, opacity_max,
                          seed, congestion)
    cfg = BuildConfigC(depth, shrink_factor, children_per_node, build_seed)
    n = C.c_uint64(0)
    nl = C.c_uint32(0)
    _check_synth(lib.lodgs_build_synthetic_tree(C.byref(spec), C.byref(cfg), None, C.byref(n), C.byref(nl)))
    t = LoDTree.empty(n.value, nl.value, shrink_factor)
    b = TreeBuffersC()
    for f in _FIELDS:
        setattr(b, f, getattr(t, f).ctypes.data_as(_FP))
    b.parent = t.parent.ctypes.data_as(C.POINTER(C.c_uint32))
    b.leaf = t.leaf.ctypes.data_as(C.POINTER(C.c_uint8))
    b.level_offsets = t.level_offsets.ctypes.data_as(C.POINTER(C.c_uint32))
    _check_synth(lib.lodgs_build_synthetic_tree(C.byref(spec), C.byref(cfg), C.byref(b), C.byref(n), C.byref(nl)))
    return t


def make_tree(seed, depth, children=8, gamma=0.5, nx=3, ny=3, congestion=1) -> LoDTree:
    """tests/unit/test_util.hpp:62-77 make_tree (reference test fixture generator)."""
    return build_synthetic_tree(nx=nx, ny=ny, seed=seed, congestion=congestion, depth=depth,
                                shrink_factor=gamma, children_per_node=children,
                                build_seed=(seed * 1099511628211 + 11) & 0xFFFFFFFFFFFFFFFF)


# ------------------------------------------------------------ GPU scene --


class _TreeShape:
    """Shape of a tree that lives only on the device (GpuScene.load)."""

    def __init__(self, n, level_offsets, shrink_factor):
        self._n = int(n)
        self.level_offsets = level_offsets
        self.shrink_factor = shrink_factor

    def node_count(self) -> int:
        return self._n


class GpuScene:
    """Device-resident copy of one LoDTree (validated once at upload)."""

    def __init__(self, tree: LoDTree, device: int = 0):
        self._lib = load_library()
        self.tree = tree
        self.device = device
        self._h = C.c_void_p(None)
        v = tree.view()
        _check(self._lib.lodgs_gpu_scene_create(C.byref(v), int(device), C.byref(self._h)))

    @classmethod
    def load(cls, path: str, device: int = 0, timing_ms=None) -> "GpuScene":
        """load_scene (scene_io.cpp:213-226) of an LDGS v1 binary file straight to
        the device (de-interleave + validate_tree on the GPU).  timing_ms: optional
        float64 array of 3 (read+H2D, de-interleave, validate+pack ms)."""
        self = cls.__new__(cls)
        self._lib = load_library()
        self.device = device
        self._h = C.c_void_p(None)
        tm = None
        if timing_ms is not None:
            assert timing_ms.dtype == np.float64 and timing_ms.size >= 3
            tm = timing_ms.ctypes.data_as(_DP)
        _check(self._lib.lodgs_gpu_scene_load(os.fsencode(path), int(device), C.byref(self._h), tm))
        n, nl, sf = C.c_uint64(0), C.c_uint32(0), C.c_float(0.0)
        _check(self._lib.lodgs_gpu_scene_info(self._h, C.byref(n), C.byref(nl), None, 0, C.byref(sf)))
        offs = np.zeros(max(1, nl.value), np.uint32)
        _check(self._lib.lodgs_gpu_scene_info(self._h, None, None, _ptr(offs), nl.value, None))
        self.tree = _TreeShape(n.value, offs[: nl.value].copy(), sf.value)
        return self

    def close(self):
        if self._h and self._h.value:
            self._lib.lodgs_gpu_scene_destroy(self._h)
            self._h = C.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def stream_ptr(self) -> int:
        p = C.c_void_p(None)
        _check(self._lib.lodgs_gpu_scene_stream(self._h, C.byref(p)))
        return int(p.value or 0)

    def memory_bytes(self) -> int:
        b = C.c_uint64(0)
        _check(self._lib.lodgs_gpu_scene_memory(self._h, C.byref(b)))
        return int(b.value)

    def reserve(self, max_pairs: int):
        _check(self._lib.lodgs_gpu_scene_reserve(self._h, int(max_pairs)))

    @staticmethod
    def params(filter: FilterConfig, mode: ShrinkMode, opts: RenderOptions) -> RenderParamsC:
        if opts.filter_mode not in ("parallel", "serial"):
            raise ValidationError("render: filter_mode is 'parallel' or 'serial'")
        if opts.blend_kernel not in _BLEND_FLAGS:
            raise ValidationError("render: blend_kernel is 'cpa', 'wsp', 'tma' or 'gather4'")
        flags = (1 if opts.exact_blend else 0) | (2 | 8 if opts.collect_kpc else 0) | \
                (4 if opts.stage_timing else 0) | (16 if opts.filter_mode == "serial" else 0) | \
                (32 if opts.output_rgb8 else 0) | _BLEND_FLAGS[opts.blend_kernel]
        return RenderParamsC(float(filter.tau_r), float(mode.tau), int(mode.kind), flags)

    def render(self, cam: Camera, filter: FilterConfig, mode: ShrinkMode,
               opts: RenderOptions = RenderOptions(), image_out: Optional[np.ndarray] = None
               ) -> RenderOutput:
        c = cam.to_c()
        p = self.params(filter, mode, opts)
        st = RenderStatsC()
        img = image_out if image_out is not None else np.empty((cam.height, cam.width, 3), np.float32)
        _check(self._lib.lodgs_gpu_render(self._h, C.byref(c), C.byref(p), _ptr(img), C.byref(st)))
        out = RenderOutput(Image(cam.width, cam.height, img), RenderStats.from_c(st))
        if opts.collect_kpc:
            out.pairs = self.read_pairs()
            out.gaussians = self.read_gaussians()
            out.kpc = self.read_kpc()
        return out

    def read_kpc(self) -> np.ndarray:
        n = C.c_uint64(0)
        _check(self._lib.lodgs_gpu_read_kpc(self._h, None, 0, C.byref(n)))
        out = np.empty(n.value, np.float64)
        _check(self._lib.lodgs_gpu_read_kpc(self._h, _ptr(out), n.value, C.byref(n)))
        return out

    def calibrate(self, views, lambda_g: float, config: FilterConfig = FilterConfig()
                  ) -> "CalibrationReport":
        """metrics.cpp:94-108 on the GPU (instrumented three-sigma renders)."""
        n = len(views)
        vc = (CameraC * max(1, n))(*[v.to_c() for v in views])
        rep = CalibrationC()
        per = np.zeros(max(1, n), np.float64)
        _check(self._lib.lodgs_gpu_calibrate(self._h, vc, n, float(lambda_g), float(config.tau_r),
                                             C.byref(rep), per.ctypes.data_as(_DP)))
        return CalibrationReport(per[: rep.n_views].copy(), rep.scene_gtc, rep.lambda_g, rep.tau,
                                 rep.n_views, list(rep.histogram))

    def render_batch(self, cams, filter: FilterConfig, mode: ShrinkMode,
                     opts: RenderOptions = RenderOptions(), host_ptrs=None):
        """Pipelined frames (lodgs_gpu_render_batch): frame i+1 computes while frame i's
        image is copied to host_ptrs[i] (raw pointers, e.g. pinned buffers)."""
        n = len(cams)
        cc = (CameraC * n)(*[c.to_c() for c in cams])
        p = self.params(filter, mode, opts)
        ptrs = (C.c_void_p * n)(*(host_ptrs if host_ptrs is not None else [None] * n))
        st = (RenderStatsC * n)()
        _check(self._lib.lodgs_gpu_render_batch(self._h, cc, n, C.byref(p), ptrs, st))
        return [RenderStats.from_c(s) for s in st]

    def render_async(self, cam: Camera, params: RenderParamsC, image_host_ptr=None):
        c = cam.to_c()
        _check(self._lib.lodgs_gpu_render_async(self._h, C.byref(c), C.byref(params), image_host_ptr))

    def render_views_async(self, cams, params: RenderParamsC, host_ptrs=None) -> None:
        """len(cams) frames as render_async calls, the LoD filter shared by each group of
        up to 4 consecutive frames (one pass over the node arrays for the group);
        host_ptrs (optional): one f32 image buffer per frame (raw pointers)."""
        n = len(cams)
        if n == 0:
            return
        cc = (CameraC * n)(*[c.to_c() for c in cams])
        ptrs = (C.c_void_p * n)(*host_ptrs) if host_ptrs is not None else None
        _check(self._lib.lodgs_gpu_render_views_async(self._h, cc, n, C.byref(params), ptrs))

    def join(self) -> None:
        """The control stream (stream_ptr) waits for every frame enqueued so far."""
        _check(self._lib.lodgs_gpu_join(self._h))

    def set_inflight(self, frames: int) -> None:
        """Frames in flight for render_async (1 to 12; default 4)."""
        _check(self._lib.lodgs_gpu_scene_set_inflight(self._h, int(frames)))

    def set_sh(self, degree: int, sh_rest=None) -> None:
        """View-dependent colour of degree 1..3 (an extension: the reference is SH0-only).
        sh_rest: float32 array (node_count, (degree+1)**2 - 1, 3), the 3DGS features_rest
        layout; a node's colour becomes max(rgb + sum_k c_k Y_k(dir), 0).  degree 0 goes
        back to SH0."""
        if degree == 0 or sh_rest is None:
            _check(self._lib.lodgs_gpu_scene_set_sh(self._h, int(degree), None, 0))
            return
        a = np.ascontiguousarray(sh_rest, dtype=np.float32)
        k = (int(degree) + 1) ** 2 - 1
        if a.ndim != 3 or a.shape[1:] != (k, 3):
            raise ValidationError(f"set_sh: sh_rest must be (nodes, {k}, 3) for degree {degree}")
        _check(self._lib.lodgs_gpu_scene_set_sh(self._h, int(degree), _ptr(a), a.shape[0]))

    def sync(self) -> RenderStats:
        st = RenderStatsC()
        _check(self._lib.lodgs_gpu_sync(self._h, C.byref(st)))
        return RenderStats.from_c(st)

    def take_totals(self, sort_bytes: bool = False):
        """(frames, sum n_selected, sum n_pairs[, sum radix-sort bytes]) since the last call."""
        f, s, p, b = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        _check(self._lib.lodgs_gpu_take_totals(self._h, C.byref(f), C.byref(s), C.byref(p),
                                               C.byref(b)))
        if sort_bytes:
            return int(f.value), int(s.value), int(p.value), int(b.value)
        return int(f.value), int(s.value), int(p.value)

    def profile(self, enable: bool):
        _check(self._lib.lodgs_gpu_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        """(frames, [mark, select, preprocess+keys, sort, blend, frame] ms summed)."""
        f = C.c_uint64(0)
        ms = np.zeros(6, np.float64)
        _check(self._lib.lodgs_gpu_profile_read(self._h, C.byref(f), ms.ctypes.data_as(_DP)))
        return int(f.value), ms

    def read_selected(self) -> np.ndarray:
        n = C.c_uint64(0)
        _check(self._lib.lodgs_gpu_read_selected(self._h, None, 0, C.byref(n)))
        out = np.empty(n.value, np.uint32)
        _check(self._lib.lodgs_gpu_read_selected(self._h, _ptr(out), n.value, C.byref(n)))
        return out

    def read_pairs(self) -> np.ndarray:
        n = C.c_uint64(0)
        _check(self._lib.lodgs_gpu_read_pairs(self._h, None, 0, C.byref(n)))
        out = np.empty(n.value, PAIR_DTYPE)
        _check(self._lib.lodgs_gpu_read_pairs(self._h, _ptr(out), n.value, C.byref(n)))
        return out

    def read_gaussians(self) -> BlendList:
        cap = self.tree.node_count()
        bl = BlendList.empty(cap)
        v = bl.view()
        _check(self._lib.lodgs_gpu_read_gaussians(self._h, C.byref(v), cap))
        return bl.truncated(int(v.n))

    def read_counts(self, n_gaussians: int, n_tiles: int):
        pg = np.zeros(max(1, n_gaussians), np.uint32)
        pt = np.zeros(max(1, n_tiles), np.uint32)
        _check(self._lib.lodgs_gpu_read_counts(self._h, _ptr(pg), n_gaussians, _ptr(pt), n_tiles))
        return pg[:n_gaussians], pt[:n_tiles]

    def read_image(self, cam: Camera) -> np.ndarray:
        img = np.empty((cam.height, cam.width, 3), np.float32)
        _check(self._lib.lodgs_gpu_read_image(self._h, _ptr(img)))
        return img

    def read_image_rgb8(self, cam: Camera) -> np.ndarray:
        """The last frame as 8-bit RGB (save_ppm quantisation, image.cpp:19-22)."""
        img = np.empty((cam.height, cam.width, 3), np.uint8)
        _check(self._lib.lodgs_gpu_read_image_rgb8(self._h, _ptr(img)))
        return img

    def set_reference_image(self) -> None:
        """Keep the last frame on the device as the psnr/ssim reference."""
        _check(self._lib.lodgs_gpu_set_reference_image(self._h))

    def compare_reference(self, want_ssim: bool = True):
        """(psnr, ssim) of the last frame against the stored reference, on the
        device (metrics.cpp:121-192); ssim is None unless requested."""
        p, q = C.c_double(0.0), C.c_double(0.0)
        _check(self._lib.lodgs_gpu_compare_reference(self._h, C.byref(p),
                                                     C.byref(q) if want_ssim else None))
        return p.value, (q.value if want_ssim else None)

    # stage entry points
    def filter(self, cam: Camera, config: FilterConfig) -> FilterResult:
        if not (config.tau_r > 0):
            raise ValidationError("filter config: tau_r > 0")
        if config.worker_count < 1:
            raise ValidationError("filter config: worker_count >= 1")
        c = cam.to_c()
        n = C.c_uint64(0)
        ps, bs = C.c_int32(0), C.c_int32(0)
        cap = self.tree.node_count()
        sel = np.empty(cap, np.uint32)
        _check(self._lib.lodgs_gpu_filter(self._h, C.byref(c), float(config.tau_r), _ptr(sel), cap,
                                          C.byref(n), C.byref(ps), C.byref(bs)))
        return FilterResult(sel[: n.value].copy(), ps.value, bs.value)

    def filter_serial(self, cam: Camera, config: FilterConfig, level_ms=None) -> FilterResult:
        """filter.cpp:60-113 on the device: one kernel + barrier per level.
        level_ms: optional float64 array (n_levels) for per-level device times."""
        if not (config.tau_r > 0):
            raise ValidationError("filter config: tau_r > 0")
        if config.worker_count < 1:
            raise ValidationError("filter config: worker_count >= 1")
        c = cam.to_c()
        n = C.c_uint64(0)
        ps, bs = C.c_int32(0), C.c_int32(0)
        cap = self.tree.node_count()
        sel = np.empty(max(1, cap), np.uint32)
        lm = None
        if level_ms is not None:
            assert level_ms.dtype == np.float64 and level_ms.size >= len(self.tree.level_offsets)
            lm = level_ms.ctypes.data_as(_DP)
        _check(self._lib.lodgs_gpu_filter_serial(self._h, C.byref(c), float(config.tau_r),
                                                 _ptr(sel), cap, C.byref(n), C.byref(ps),
                                                 C.byref(bs), lm))
        return FilterResult(sel[: n.value].copy(), ps.value, bs.value)

    def mark(self, cam: Camera, tau_r: float, begin: int = 0, end: Optional[int] = None,
             vis=None, qpass=None, radius=None):
        n = self.tree.node_count()
        end = n if end is None else end
        vis = np.zeros(n, np.uint8) if vis is None else vis
        qpass = np.zeros(n, np.uint8) if qpass is None else qpass
        c = cam.to_c()
        _check(self._lib.lodgs_gpu_mark(self._h, C.byref(c), begin, end, float(tau_r), _ptr(vis),
                                        _ptr(qpass), _ptr(radius)))
        return vis, qpass, radius

    def prepare(self, cam: Camera, selected: np.ndarray, mode: ShrinkMode) -> BlendList:
        sel = np.ascontiguousarray(selected, np.uint32)
        bl = BlendList.empty(max(1, sel.shape[0]))
        v = bl.view()
        c = cam.to_c()
        _check(self._lib.lodgs_gpu_prepare(self._h, C.byref(c), _ptr(sel), sel.shape[0],
                                           int(mode.kind), float(mode.tau), C.byref(v)))
        return bl.truncated(int(v.n))


# ---------------------------------------- reference-shaped free functions --

_scene_cache: dict = {}


def _scene_for(tree: LoDTree, device: int = 0) -> GpuScene:
    """The compatibility path of SURVEY.md 8(b): cache the device copy keyed on the
    tree's array identities (the tree is immutable while in use)."""
    key = (id(tree), tree.mean_x.ctypes.data, tree.node_count(), device)
    s = _scene_cache.get(key)
    if s is None or s.tree is not tree:
        _scene_cache.clear()
        s = GpuScene(tree, device)
        _scene_cache[key] = s
    return s


def render(tree: LoDTree, cam: Camera, filter: FilterConfig, mode: ShrinkMode,
           opts: RenderOptions = RenderOptions()) -> RenderOutput:
    """rasterizer.hpp:106-108 on the GPU (device copy of the tree cached)."""
    if mode.kind != ShrinkMode.THREE_SIGMA and not (0.0 < mode.tau < 1.0):
        raise ValidationError("render: shrink tau in (0,1); adaptive needs calibration first")
    return _scene_for(tree).render(cam, filter, mode, opts)


def filter_parallel(tree: LoDTree, cam: Camera, config: FilterConfig) -> FilterResult:
    """filter.hpp:42-43 -- passes = barriers = 2."""
    return _scene_for(tree).filter(cam, config)


def _image_array(img) -> np.ndarray:
    a = img.rgb if isinstance(img, Image) else img
    return np.ascontiguousarray(a, np.float32)


def _metrics(a, b, want_psnr, want_ssim):
    x, y = _image_array(a), _image_array(b)
    if x.shape != y.shape or x.ndim != 3 or x.shape[2] != 3:
        raise ValidationError("psnr: image dimensions differ" if want_psnr else
                              "ssim: image dimensions differ")
    h, w = x.shape[0], x.shape[1]
    p, q = C.c_double(0.0), C.c_double(0.0)
    _check(load_library().lodgs_gpu_image_metrics(_ptr(x), _ptr(y), w, h,
                                                  C.byref(p) if want_psnr else None,
                                                  C.byref(q) if want_ssim else None))
    return p.value, q.value


class PinnedImage:
    """An f32 RGB image in pinned host memory (lodgs_gpu_host_alloc): a synchronous render
    into it copies each band of rows while the next band blends (pageable memory gets one
    copy after the blend).  Use as a context manager; .rgb is the (H, W, 3) array."""

    def __init__(self, width: int, height: int):
        self._lib = load_library()
        n = int(width) * int(height) * 3
        p = C.c_void_p()
        _check(self._lib.lodgs_gpu_host_alloc(n * 4, C.byref(p)))
        self._p = p.value
        self.rgb = np.ctypeslib.as_array((C.c_float * n).from_address(self._p)).reshape(
            int(height), int(width), 3)

    def close(self) -> None:
        if self._p:
            self.rgb = None
            self._lib.lodgs_gpu_host_free(self._p)
            self._p = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def psnr(a, b) -> float:
    """metrics.hpp psnr (metrics.cpp:121-132) on the device; +inf if identical."""
    return _metrics(a, b, True, False)[0]


def ssim(a, b) -> float:
    """metrics.hpp ssim (metrics.cpp:136-192): mean 11x11 Gaussian-window SSIM
    over the three channels, on the device."""
    return _metrics(a, b, False, True)[1]


def filter_serial(tree: LoDTree, cam: Camera, config: FilterConfig) -> FilterResult:
    """filter.hpp:37-38 -- level-wise; passes = barriers = levels descended."""
    return _scene_for(tree).filter_serial(cam, config)


def prepare_gaussians(tree: LoDTree, cam: Camera, selected, mode: ShrinkMode) -> BlendList:
    """rasterizer.hpp:55-57."""
    return _scene_for(tree).prepare(cam, selected, mode)


def bin_to_tiles(lst: BlendList, grid: TileGrid, width: int, height: int) -> np.ndarray:
    """rasterizer.hpp:59-62 -- reference emission order."""
    lib = load_library()
    v = lst.view()
    n = C.c_uint64(0)
    _check(lib.lodgs_gpu_bin_to_tiles(C.byref(v), int(width), int(height), None, 0, C.byref(n)))
    out = np.empty(n.value, PAIR_DTYPE)
    _check(lib.lodgs_gpu_bin_to_tiles(C.byref(v), int(width), int(height), _ptr(out), n.value,
                                      C.byref(n)))
    return out


def sort_pairs(pairs: np.ndarray) -> None:
    """rasterizer.hpp:64-65 -- (tile, depth) stable order, in place."""
    if pairs.dtype != PAIR_DTYPE or not pairs.flags.c_contiguous:
        raise ValidationError("sort_pairs: expects a contiguous PAIR_DTYPE array")
    _check(load_library().lodgs_gpu_sort_pairs(_ptr(pairs), pairs.shape[0]))


def alpha_blend(sorted_pairs: np.ndarray, lst: BlendList, grid: TileGrid, width: int, height: int,
                workers: int = 1, exact: bool = False, blend_kernel: str = "cpa") -> Image:
    """rasterizer.hpp:67-71 (kpc collection is not part of this stage on the GPU)."""
    sp = np.ascontiguousarray(sorted_pairs, PAIR_DTYPE)
    img = np.empty((height, width, 3), np.float32)
    v = lst.view()
    flags = (1 if exact else 0) | _BLEND_FLAGS[blend_kernel]
    _check(load_library().lodgs_gpu_alpha_blend(_ptr(sp), sp.shape[0], C.byref(v), int(width),
                                                int(height), flags, _ptr(img)))
    return Image(width, height, img)


def calibrate(tree: LoDTree, views, lambda_g: float, filter: FilterConfig = FilterConfig()
              ) -> CalibrationReport:
    """metrics.hpp:73-75 calibrate -> CalibrationReport (tau = lambda_g / mean view GTC)."""
    return _scene_for(tree).calibrate(views, lambda_g, filter)
