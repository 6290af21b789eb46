/* lodgs_gpu.h -- C ABI of the B200-native FilterGS per-frame renderer.
 *
 * This is the drop-in boundary for the reference's per-frame hot path,
 *     lodgs::render(tree, cam, FilterConfig, ShrinkMode, RenderOptions)
 *     (/root/reference/proj/include/lodgs/rasterizer.hpp:106-108, body
 *      proj/src/rasterizer.cpp:167-213)
 * and for its stage functions filter_parallel / prepare_gaussians /
 * bin_to_tiles / sort_pairs / alpha_blend (filter.hpp:42-43,
 * rasterizer.hpp:55-71).  Plain pointers and sizes only; no C++ or torch
 * types.  The reference-side C++ shim (integration/rasterizer_b200.cpp, the
 * maintainer-added lodgs::render of INTEGRATION.md, linked and run against the
 * reference library by tests/test_gpu_integration.py) and the Python host module
 * (paper_2603_23891_b200/lodgs.py) both sit on top of these entry points.
 *
 * Every compute entry point runs hand-written sm_100a CUDA kernels; there is
 * no CPU fallback.  Without a usable CUDA device the compute calls return
 * LODGS_ERR_CUDA and lodgs_gpu_last_error() says why.
 *
 * Status codes mirror the reference CLI's exit codes (cli.cpp:28-29):
 * 0 ok, 2 validation/format (ValidationError / FormatError), 3 I/O (IoError).
 * 4 and 5 are new: CUDA runtime failure and internal error.
 */
#ifndef LODGS_GPU_H
#define LODGS_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LODGS_GPU_ABI_VERSION 1

#if defined(__GNUC__)
#define LODGS_API __attribute__((visibility("default")))
#else
#define LODGS_API
#endif

enum lodgs_status {
    LODGS_OK = 0,
    LODGS_ERR_VALIDATION = 2, /* core.hpp:91-93 ValidationError / FormatError */
    LODGS_ERR_IO = 3,         /* core.hpp:96-98 IoError */
    LODGS_ERR_CUDA = 4,
    LODGS_ERR_INTERNAL = 5
};

/* scene.hpp:76-82 Camera.  `znear`/`zfar` are the reference's near/far. */
typedef struct lodgs_camera {
    uint32_t width, height;
    double fx, fy, cx, cy;
    double rotation[9]; /* world->camera, row-major */
    double translation[3];
    double znear, zfar;
} lodgs_camera;

/* scene.hpp:29-74 LoDTree (level-major SoA arena), borrowed for the call. */
typedef struct lodgs_tree_view {
    uint64_t n_nodes;
    const float *mean_x, *mean_y, *mean_z;
    const float *scale_x, *scale_y, *scale_z;
    const float *quat_w, *quat_x, *quat_y, *quat_z;
    const float *opacity;
    const float *color_r, *color_g, *color_b;
    const uint32_t *parent; /* 0xFFFFFFFF = root (core.hpp:15) */
    const uint8_t *leaf;
    const uint32_t *level_offsets;
    uint32_t n_levels;
    float shrink_factor;
} lodgs_tree_view;

/* rasterizer.hpp:16-24 ShrinkMode::Kind */
enum lodgs_shrink_kind {
    LODGS_SHRINK_THREE_SIGMA = 0,
    LODGS_SHRINK_FIXED = 1,   /* tau = 1/255 */
    LODGS_SHRINK_ADAPTIVE = 2 /* tau from calibration */
};

/* Render flags (no reference equivalent except KEEP_PAIRS ~ collect_kpc). */
enum lodgs_render_flags {
    LODGS_RENDER_EXACT_BLEND = 1u,  /* FP64 blend with the reference exp_mx: bit-exact image */
    LODGS_RENDER_KEEP_PAIRS = 2u,   /* keep sorted pairs + gaussians readable after the frame */
    LODGS_RENDER_STAGE_TIMING = 4u, /* CUDA-event stage timers into lodgs_render_stats */
    LODGS_RENDER_COLLECT_KPC = 8u,  /* RenderOptions::collect_kpc: per-pair kpc, exact blend */
    LODGS_RENDER_FILTER_SERIAL = 16u, /* RenderOptions::filter_mode = serial (filter.cpp:60-113) */
    LODGS_RENDER_OUTPUT_RGB8 = 32u, /* host images are W*H*3 bytes, save_ppm's quantisation
                                       (image.cpp:19-22), 1/4 of the PCIe bytes */
    /* Fast-blend kernel (all certified-identical).  Default (no flag):
     * k_blend_cpa, the fastest measured on the BASELINE configs. */
    LODGS_RENDER_BLEND_TMA = 64u,   /* k_blend_tma: the sort writes a 48 B record per pair,
                                       each tile's records stream into shared memory with
                                       cp.async.bulk (TMA) */
    LODGS_RENDER_BLEND_GATHER4 = 128u, /* k_blend_g4: TMA tile::gather4 of the slot-indexed
                                          records, no record pass */
    LODGS_RENDER_BLEND_CPA = 256u, /* k_blend_cpa (the default): one producer warp streams
                                      the records with per-lane cp.async into a 20-stage ring,
                                      the 8 consumer warps cull against their 8x4 blocks */
    LODGS_RENDER_BLEND_WSP = 512u  /* k_blend_wsp (round-1 default): two producer warps
                                      gather, cull and hand per-block hit lists over a
                                      5-stage ring */
};

/* FilterConfig (filter.hpp:11-14) + ShrinkMode (rasterizer.hpp:16-24). */
typedef struct lodgs_render_params {
    double tau_r;        /* pixel radius threshold, > 0 */
    double tau;          /* opacity threshold for fixed/adaptive, in (0,1) */
    int32_t shrink_kind; /* lodgs_shrink_kind */
    uint32_t flags;      /* lodgs_render_flags */
} lodgs_render_params;

/* RenderStats (rasterizer.hpp:73-84) plus the device-side counts. */
typedef struct lodgs_render_stats {
    uint64_t n_selected;  /* filter survivors */
    uint64_t n_gaussians; /* projected (selected minus near-plane drops) */
    uint64_t n_pairs;     /* N_P, gaussian-tile pairs */
    int32_t filter_passes, filter_barriers; /* 2 / 2 as filter_parallel */
    double t_calc_ms, t_sync_ms, t_prepr_ms, t_sort_ms, t_alpha_ms;
    uint32_t big_tiles; /* tiles sorted by the large-segment path */
    uint32_t kernel_launches;
} lodgs_render_stats;

/* tiles.hpp:23-28 TilePair */
typedef struct lodgs_tile_pair {
    uint32_t tile;
    float depth;
    uint32_t gaussian;
} lodgs_tile_pair;

/* rasterizer.hpp:36-51 BlendList, caller-owned arrays (capacity >= n). */
typedef struct lodgs_blend_list {
    uint64_t n;
    double *mean_x, *mean_y;
    double *conic_a, *conic_b, *conic_c;
    double *opacity;
    double *col_r, *col_g, *col_b;
    double *radius;
    float *depth;
    uint32_t *node;
} lodgs_blend_list;

typedef struct lodgs_gpu_scene lodgs_gpu_scene;

/* ---------------------------------------------------------------- misc -- */
LODGS_API const char *lodgs_gpu_last_error(void);
LODGS_API int lodgs_gpu_abi_version(void);
LODGS_API int lodgs_gpu_device_count(int *count);

/* ------------------------------------------------- host-side utilities -- */
/* scene.cpp:89-165 validate_tree; *n_violations = number of rule breaks.
 * msg (optional) receives the same text require_valid would throw. */
LODGS_API int lodgs_validate_tree(const lodgs_tree_view *tree, uint64_t *n_violations, char *msg,
                        size_t msg_cap);
/* scene.cpp:167-199 validate_camera. */
LODGS_API int lodgs_validate_camera(const lodgs_camera *cam, uint64_t *n_violations, char *msg,
                          size_t msg_cap);
/* projection.cpp:11-38 CameraGeom::make, 44 doubles in CameraGeom order. */
LODGS_API int lodgs_camera_geom(const lodgs_camera *cam, double out44[44]);
/* ---------------------------------------------------------- GPU scenes -- */
/* Validates the tree once (the reference re-validates every frame,
 * rasterizer.cpp:170) and uploads it to `device`.  The scene owns one CUDA
 * stream; calls on one scene are serialised by the caller. */
LODGS_API int lodgs_gpu_scene_create(const lodgs_tree_view *tree, int device, lodgs_gpu_scene **out);
/* load_scene (scene_io.cpp:213-226) of an LDGS v1 binary file straight into a
 * device scene: the payload streams through pinned buffers to the device, where
 * kernels de-interleave it (scene_io.cpp:90-116) and run validate_tree's
 * per-node rules (scene.cpp:122-162) once.  Errors as the reference: IoError
 * (cannot open) -> LODGS_ERR_IO; FormatError (bad magic, unsupported version,
 * truncated ... reading <section>) and ValidationError -> LODGS_ERR_VALIDATION.
 * JSON scenes are refused (load them on the host, then lodgs_gpu_scene_create).
 * timing_ms (nullable, 3): read+H2D, de-interleave, validate+pack wall times. */
LODGS_API int lodgs_gpu_scene_load(const char *path, int device, lodgs_gpu_scene **out,
                         double *timing_ms);
/* Shape of a device scene (for scenes loaded from files): node count, level
 * begins (capacity cap), shrink factor; any output may be NULL. */
LODGS_API int lodgs_gpu_scene_info(lodgs_gpu_scene *scene, uint64_t *n_nodes, uint32_t *n_levels,
                         uint32_t *level_offsets, uint32_t cap, float *shrink_factor);
LODGS_API int lodgs_gpu_scene_destroy(lodgs_gpu_scene *scene);
/* The scene's cudaStream_t, for callers that time on it with CUDA events. */
LODGS_API int lodgs_gpu_scene_stream(lodgs_gpu_scene *scene, void **stream);
/* Pre-sizes the pair buffer (bytes are 16 * max_pairs). Grows on demand otherwise. */
LODGS_API int lodgs_gpu_scene_reserve(lodgs_gpu_scene *scene, uint64_t max_pairs);
/* Device bytes held by the scene. */
LODGS_API int lodgs_gpu_scene_memory(lodgs_gpu_scene *scene, uint64_t *bytes);

/* One frame, synchronous, the reference render() contract: filter ->
 * preprocess(+shrink) -> key duplication -> sort -> blend.  image_host
 * (nullable) receives W*H*3 interleaved RGB f32 (Image, image.hpp:10-23);
 * pinned memory from lodgs_gpu_host_alloc makes the copy DMA-direct. */
LODGS_API int lodgs_gpu_render(lodgs_gpu_scene *scene, const lodgs_camera *cam,
                     const lodgs_render_params *params, float *image_host,
                     lodgs_render_stats *stats);

/* n frames through the render() contract, pipelined: frame i+1 is computed
 * while frame i's image is copied to images_host[i] on a second stream
 * (double-buffered device images).  images_host[i] may repeat a buffer only
 * if the caller does not need frame i's image after frame i+2 starts.
 * stats (nullable) receives n entries.  Overflowing frames are re-rendered. */
LODGS_API int lodgs_gpu_render_batch(lodgs_gpu_scene *scene, const lodgs_camera *cams,
                                     uint64_t n, const lodgs_render_params *params,
                                     float *const *images_host, lodgs_render_stats *stats);

/* Enqueue one frame on the scene stream and return without synchronising.
 * Sizes stay on the device; an undersized pair buffer is reported (and
 * grown) by the next lodgs_gpu_sync, which then returns LODGS_ERR_INTERNAL
 * with "overflow" so the caller re-renders. image_host (nullable) is filled
 * by an async D2H copy on the same stream. */
LODGS_API int lodgs_gpu_render_async(lodgs_gpu_scene *scene, const lodgs_camera *cam,
                           const lodgs_render_params *params, float *image_host);
/* n frames enqueued like n lodgs_gpu_render_async calls, with the LoD filter shared
 * by each group of V = min(4, frames in flight / 2) consecutive frames: one pass over
 * the node arrays decides every node for all the group's views (SURVEY.md 8(e)'s
 * multi-view option; filter.cpp:115-150 per view); groups rotate over the in-flight / V
 * disjoint sets of V contexts.  Each frame's outputs equal its single-view render bit for bit.
 * Frames with per-frame-only flags (stage timing, serial filter, collect_kpc, keep
 * pairs), mixed resolutions or fewer than 4 frames in flight fall back to per-frame
 * enqueues. */
LODGS_API int lodgs_gpu_render_views_async(lodgs_gpu_scene *scene, const lodgs_camera *cams,
                                           uint64_t n, const lodgs_render_params *params,
                                           float *const *images_host);
/* Waits for every in-flight frame; stats (nullable) = the last frame's. */
LODGS_API int lodgs_gpu_sync(lodgs_gpu_scene *scene, lodgs_render_stats *stats);
/* Frames in flight for lodgs_gpu_render_async: 1 to 12 (default 4) -- consecutive
 * frames rotate over the scene and up to three twin contexts (own stream and
 * per-frame buffers over the same device tree), so one frame's latency-bound
 * kernels overlap the others'.  All fork from the scene's control stream
 * (lodgs_gpu_scene_stream): a frame starts after the work already enqueued
 * there (e.g. a timing event). */
LODGS_API int lodgs_gpu_scene_set_inflight(lodgs_gpu_scene *scene, int frames);

/* View-dependent colour, spherical harmonics of degree 1..3 (BASELINE configs[1],
 * "SH deg 3"; an extension: the reference is SH0-only, scene.hpp:15-24, so
 * these colours have no reference to match -- DESIGN.md 3.9).  sh_rest holds, per node,
 * K = (degree+1)^2 - 1 coefficients x 3 channels (K-major, the 3DGS features_rest layout),
 * n_nodes rows.  A node's colour becomes max(rgb + sum_k c_k Y_k(d), 0), d the unit
 * direction from the camera centre to the node's mean, rgb its SH0 colour; with all
 * coefficients zero every frame equals the SH0 frame bit for bit.  degree 0 (sh_rest
 * ignored) goes back to SH0.  2: degree outside 0..3, n_nodes != the scene's node count,
 * or a non-finite coefficient. */
LODGS_API int lodgs_gpu_scene_set_sh(lodgs_gpu_scene *scene, int degree, const float *sh_rest,
                                     uint64_t n_nodes);
/* Makes the control stream wait for every frame enqueued so far (no host sync):
 * record a timing event on the control stream after this. */
LODGS_API int lodgs_gpu_join(lodgs_gpu_scene *scene);
/* Sum of n_selected / n_pairs over frames since the last call (device counters);
 * sum_sort_bytes (nullable): the SURVEY 8(d) radix-sort bytes of those frames,
 * (24 B x non-uniform 8-bit digits of the reference key + 8 B) per pair. */
LODGS_API int lodgs_gpu_take_totals(lodgs_gpu_scene *scene, uint64_t *frames, uint64_t *sum_selected,
                          uint64_t *sum_pairs, uint64_t *sum_sort_bytes);

/* Per-stage CUDA-event profiling of every enqueued frame, without host sync.
 * enable=1 starts (and clears) collection, enable=0 stops it.  read() syncs
 * and returns, summed over the collected frames, the device time of
 * stage_ms[0] filter mark (K1), [1] filter select (K2), [2] preprocess +
 * tile offsets + key duplication (K3/K4), [3] per-tile sort (K5),
 * [4] blend (K6), [5] whole frame. */
LODGS_API int lodgs_gpu_profile(lodgs_gpu_scene *scene, int enable);
LODGS_API int lodgs_gpu_profile_read(lodgs_gpu_scene *scene, uint64_t *frames, double stage_ms[6]);

/* Readbacks of the last frame (after lodgs_gpu_sync / lodgs_gpu_render). */
LODGS_API int lodgs_gpu_read_image(lodgs_gpu_scene *scene, float *out);
LODGS_API int lodgs_gpu_image_device_ptr(lodgs_gpu_scene *scene, const float **dev_ptr);
LODGS_API int lodgs_gpu_read_selected(lodgs_gpu_scene *scene, uint32_t *out, uint64_t cap, uint64_t *n);
/* Sorted (tile, depth, gaussian) pairs: needs LODGS_RENDER_KEEP_PAIRS. */
LODGS_API int lodgs_gpu_read_pairs(lodgs_gpu_scene *scene, lodgs_tile_pair *out, uint64_t cap,
                         uint64_t *n);
/* The projected BlendList (FP64 fields): needs LODGS_RENDER_KEEP_PAIRS. */
LODGS_API int lodgs_gpu_read_gaussians(lodgs_gpu_scene *scene, lodgs_blend_list *out, uint64_t cap);
/* Per-pair kpc of the last frame in sorted-pair order (needs LODGS_RENDER_COLLECT_KPC):
 * RenderOutput::kpc (rasterizer.hpp:86-96), bit-identical to blend_scalar.cpp:16-54. */
LODGS_API int lodgs_gpu_read_kpc(lodgs_gpu_scene *scene, double *out, uint64_t cap, uint64_t *n);

/* metrics.hpp:44-54 CalibrationReport. */
typedef struct lodgs_calibration {
    double tau;        /* lambda_g / scene_gtc */
    double scene_gtc;  /* mean of the per-view GTCs */
    double lambda_g;
    uint32_t n_views;  /* views that produced pairs */
    uint64_t histogram[5];
} lodgs_calibration;

/* calibrate (metrics.cpp:94-108): per view an instrumented three-sigma render
 * (exact blend + kpc), tile GTCs, view GTC (metrics.cpp:18-42); views without
 * pairs are skipped; tau = lambda_g / mean.  per_view (nullable) receives the
 * used views' GTCs (capacity n_views). */
LODGS_API int lodgs_gpu_calibrate(lodgs_gpu_scene *scene, const lodgs_camera *views,
                                  uint32_t n_views, double lambda_g, double tau_r,
                                  lodgs_calibration *out, double *per_view);

/* Per-gaussian tile counts (bin_to_tiles multiplicity) and per-tile pair counts. */
LODGS_API int lodgs_gpu_read_counts(lodgs_gpu_scene *scene, uint32_t *per_gaussian, uint64_t cap_g,
                          uint32_t *per_tile, uint64_t cap_t);

/* -------------------------------------------------- stage entry points -- */
/* filter_parallel (filter.cpp:115-150): selected ascending, passes = barriers = 2. */
LODGS_API int lodgs_gpu_filter(lodgs_gpu_scene *scene, const lodgs_camera *cam, double tau_r,
                     uint32_t *selected, uint64_t cap, uint64_t *n_selected, int32_t *passes,
                     int32_t *barriers);
/* filter_serial (filter.cpp:60-113): level-wise traversal, one kernel and one
 * barrier per level (the paper's serial baseline); selected
 * ascending; passes = barriers = levels with an active node.  level_ms
 * (nullable, n_levels entries) receives each level's device time. */
LODGS_API int lodgs_gpu_filter_serial(lodgs_gpu_scene *scene, const lodgs_camera *cam, double tau_r,
                            uint32_t *selected, uint64_t cap, uint64_t *n_selected,
                            int32_t *passes, int32_t *barriers, double *level_ms);
/* MarkFn contract (kernels.hpp:47-52) over [begin, end): vis, qpass and
 * (nullable) the FP64 screen radius, bit-identical to mark_scalar. */
LODGS_API int lodgs_gpu_mark(lodgs_gpu_scene *scene, const lodgs_camera *cam, uint64_t begin, uint64_t end,
                   double tau_r, uint8_t *vis, uint8_t *qpass, double *radius);
/* prepare_gaussians (rasterizer.cpp:48-73); out arrays need n_sel capacity. */
LODGS_API int lodgs_gpu_prepare(lodgs_gpu_scene *scene, const lodgs_camera *cam, const uint32_t *selected,
                      uint64_t n_sel, int32_t shrink_kind, double tau, lodgs_blend_list *out);
/* bin_to_tiles (rasterizer.cpp:75-98) in the reference's emission order.
 * out == NULL: only *n_pairs is computed. */
LODGS_API int lodgs_gpu_bin_to_tiles(const lodgs_blend_list *list, int width, int height,
                           lodgs_tile_pair *out, uint64_t cap, uint64_t *n_pairs);
/* sort_pairs (rasterizer.cpp:100-135): stable (tile, depth) order, in place. */
LODGS_API int lodgs_gpu_sort_pairs(lodgs_tile_pair *pairs, uint64_t n);
/* alpha_blend (rasterizer.cpp:137-165) of sorted pairs; flags may hold
 * LODGS_RENDER_EXACT_BLEND. image receives W*H*3 floats. */
LODGS_API int lodgs_gpu_alpha_blend(const lodgs_tile_pair *sorted, uint64_t n, const lodgs_blend_list *list,
                          int width, int height, uint32_t flags, float *image);

/* ------------------------------------------- image metrics, 8-bit output -- */
/* The current image as 8-bit RGB with save_ppm's quantisation (image.cpp:19-22:
 * clamp to [0,1], floor(v*255+0.5)); out receives W*H*3 bytes (1/4 of the f32
 * image's PCIe traffic). */
LODGS_API int lodgs_gpu_read_image_rgb8(lodgs_gpu_scene *scene, uint8_t *out);
/* Keep the current image on the device as the comparison reference (bench.cpp:
 * the first combination's frames are the reference of the others). */
LODGS_API int lodgs_gpu_set_reference_image(lodgs_gpu_scene *scene);
/* psnr / ssim (metrics.cpp:121-192) of the current image against the stored
 * reference, computed on the device; either output may be NULL.  Same
 * dimensions required (ValidationError otherwise); psnr = +inf for identical
 * images.  Per-window SSIM follows the reference's operation order; the sums
 * over pixels / windows are re-associated (deterministic, not bit-equal). */
LODGS_API int lodgs_gpu_compare_reference(lodgs_gpu_scene *scene, double *psnr, double *ssim);
/* psnr / ssim of two host images (W*H*3 floats) on the current device. */
LODGS_API int lodgs_gpu_image_metrics(const float *a, const float *b, int width, int height,
                            double *psnr, double *ssim);

/* ----------------------------------------------------------- utilities -- */
/* Pinned host memory for zero-staging image readback. */
LODGS_API int lodgs_gpu_host_alloc(uint64_t bytes, void **ptr);
LODGS_API int lodgs_gpu_host_free(void *ptr);

#ifdef __cplusplus
}
#endif
#endif /* LODGS_GPU_H */
