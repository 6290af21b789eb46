// launch.h -- host-side launch wrappers for the sm_100a kernels.
// Everything here is enqueued on the caller's stream; nothing synchronises.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "blend_rec.cuh"
#include "common.cuh"

namespace fgs {

// Device copy of one LoDTree (scene.hpp:29-74), laid out for the access
// patterns of the frame.  The filter streams one 16-byte record per node
// (mean + max scale: all a frustum test reads) and the parent index; only the
// internal region [0, leaf_begin) -- 1/8 of a K=8 tree -- also carries the
// scales and quaternion its EWA radius needs.  The preprocess gathers one
// 64-byte AoS record per selected node.
struct DevTree {
    uint64_t n = 0;
    const float4* geo = nullptr;     // (mx, my, mz, max(sx, sy, sz)), padded to 256 nodes
    const float4* iscale = nullptr;  // (sx, sy, sz, leaf ? 1 : 0) for [0, leaf_begin)
    const float4* iquat = nullptr;   // (w, x, y, z) for [0, leaf_begin)
    const uint32_t* parent = nullptr;  // padded to 256 nodes with kRootParent
    const SplatRec* splat = nullptr;
    // optional SH rest coefficients (lodgs_gpu_scene_set_sh): sh_k per channel
    // (3 / 8 / 15 for degree 1 / 2 / 3, 0: SH0), per node 3 sh_k floats K-major,
    // padded to whole float4s (sh_stride of them)
    const float4* sh = nullptr;
    int sh_k = 0, sh_stride = 0;
    // Nodes [leaf_begin, n) are all leaves (leaf_begin a multiple of 1024, or n).
    uint64_t leaf_begin = 0;
    // max_i (|mx| + |my| + |mz|) over the tree (rounded up): the FP32 leaf
    // frustum pre-test's magnitude bound
    double max_l1 = 0.0;
};

// ---- filter (filter.cpp:115-150) ----
// kernels enqueued per frame besides the filter's filter_launches(n): zero,
// preprocess, tile offsets (+ run totals), emit, tile sort, big-tile sort, then
// blend_launches() for the blend
constexpr int kLaunchesPerFrame = 6;
constexpr int kMarkBlock = 256;
constexpr int kSelectBlock = 256;
#ifndef SELECT_ITEMS
#define SELECT_ITEMS 8
#endif
constexpr int kSelectItems = SELECT_ITEMS;  // nodes per thread -> 2048-node tiles
// k_select_internal's per-warp survivor sum covers 8 words (4 and 8 measured alike)
static_assert(kSelectItems >= 1 && kSelectItems <= 8, "select: at most 8 nodes per thread");
// bitmask words, rounded up to whole 8192-node compaction tiles
inline uint64_t bit_words(uint64_t n) { return (n + 8191) / 8192 * 256; }
inline uint32_t select_tiles(uint64_t n) {
    return uint32_t((n + uint64_t(kSelectBlock) * kSelectItems - 1) /
                    (uint64_t(kSelectBlock) * kSelectItems));
}
// The whole filter, four kernels: F1 internal marks, F2 internal chain walks,
// F3 fused leaf pass, F4 ordered compaction into `selected` (n_selected lands
// in cnt).  `mid` (optional) is recorded between F2 and F3.  tile_count: zeroed per frame, filter_status_entries(n) words.
// clk (nullable): per-kernel device times (FrameCounters::clock) for the
// T_calcu / T_synch split of the stage timers.
void launch_filter(const Geom& g, const DevTree& t, double tau_r, uint32_t* cand_bits,
                   uint32_t* qint_bits, uint32_t* tile_count, uint32_t* selected,
                   FrameCounters* cnt, cudaStream_t s, cudaEvent_t mid = nullptr,
                   FilterClock* clk = nullptr);
// Multi-view filter: up to kMaxViews views of one tree in one pass over the node
// arrays (F1 and F3 shared, F2 and F4 per view); each view's outputs equal
// launch_filter's for that view.  The per-view buffers must be zeroed as for
// launch_filter (tile counts, counters).
constexpr int kMaxViews = 4;
struct ViewSet {
    int n = 0;
    Geom g[kMaxViews];
    uint32_t* cand[kMaxViews] = {};
    uint32_t* qint[kMaxViews] = {};
    uint32_t* tile_count[kMaxViews] = {};
    uint32_t* selected[kMaxViews] = {};
    FrameCounters* cnt[kMaxViews] = {};
};
void launch_filter_views(const ViewSet& views, const DevTree& t, double tau_r, cudaStream_t s);
// Serial (level-wise) filter, filter.cpp:60-113: one kernel per level, then
// the ordered compaction.  level_flag[n_levels] (zeroed) marks the levels with
// an active node; level_events (nullable, n_levels + 1) time the levels.
void launch_filter_serial(const Geom& g, const DevTree& t, double tau_r,
                          const uint64_t* level_begin, int n_levels, uint32_t* sel_bits,
                          uint32_t* exp_bits, uint32_t* tile_count, unsigned* level_flag,
                          uint32_t* selected, FrameCounters* cnt, cudaEvent_t* level_events,
                          cudaStream_t s, FilterClock* clk = nullptr);
// per-tile survivor counters the filter needs for an n-node tree
uint32_t filter_status_entries(uint64_t n);
// kernels launch_filter enqueues for an n-node tree (4, or 5 with the tile-count scan)
int filter_launches(uint64_t n);
void launch_mark_debug(const Geom& g, const DevTree& t, uint64_t begin, uint64_t end,
                       double tau_r, uint8_t* vis, uint8_t* qpass, double* radius,
                       cudaStream_t s);

// ---- preprocess (rasterizer.cpp:36-98) ----
constexpr int kPrepBlock = 256;
struct PrepOut {
    Gauss64* g64;
    Gauss32* g32;
    GaussEmit* emit;
    GaussCol64* col64;     // nullable: only for the exact blend
    uint32_t* tile_count;  // n_tiles, zeroed per frame
    // nullable: each CTA's nonzero (tile, count) entries of its shared tile
    // histogram (grid x n_tiles capacity) and their number, so K4 reserves its
    // runs without recounting
    uint2* tile_lists = nullptr;
    uint32_t* tile_list_len = nullptr;
};
constexpr int kHistMaxTiles = 12288;  // shared-memory tile histograms up to 48 KB
constexpr int16_t kDropped = -32768;  // GaussEmit::ty0 of a slot dropped by project()
void launch_preprocess(const Geom& g, const DevTree& t, const uint32_t* selected,
                       uint64_t max_selected, int shrink_kind, double tau, int tiles_x,
                       int tiles_y, PrepOut out, FrameCounters* cnt, int grid, cudaStream_t s,
                       bool known_visible = false);
// SH degree 1..3 colours of the kept slots (after launch_preprocess; no-op without SH)
void launch_sh_colour(const Geom& g, const DevTree& t, const GaussEmit* emit, Gauss32* g32,
                      GaussCol64* col64, const FrameCounters* cnt, int grid, cudaStream_t s);
// Turns the per-tile counts into offsets[n_tiles+1] and per-tile write cursors,
// lists the tiles whose segment exceeds the in-shared-memory sort capacity, and
// writes order[n_tiles]: tiles heaviest-first (log2 buckets) for the per-tile grids.
// With `totals`, also accumulates the per-run frame/selected/pair totals; with
// `log`, copies the frame's final counters there (device-side batch log).
void launch_tile_offsets(const uint32_t* tile_count, int n_tiles, uint32_t* offsets,
                         uint32_t* cursor, uint32_t* big_list, uint32_t* order,
                         FrameCounters* cnt, uint64_t pair_cap, cudaStream_t s,
                         RunTotals* totals = nullptr, FrameCounters* log = nullptr);
// Key duplication: one key per (gaussian, overlapped tile) scattered into the
// tile's bucket; key = depth_bits << 32 | gaussian.
void launch_emit_keys(const GaussEmit* emit, const FrameCounters* cnt, int tiles_x, int n_tiles,
                      uint32_t* cursor, unsigned long long* keys, int grid, cudaStream_t s,
                      const uint2* tile_lists = nullptr, const uint32_t* tile_list_len = nullptr);
// Readbacks: slot -> BlendList index map, and slot-indexed records compacted
// into BlendList order.
void launch_slot_map(const GaussEmit* emit, uint64_t n, unsigned long long* status,
                     FrameCounters* cnt, uint32_t* g_of_slot, uint32_t* slot_of_g, int grid,
                     cudaStream_t s);
void launch_compact_records(const uint32_t* slot_of_g, uint64_t n_g, const Gauss64* g64,
                            const Gauss32* g32, const GaussEmit* emit, Gauss64* o64, Gauss32* o32,
                            GaussEmit* oe, cudaStream_t s);

// ---- sort (rasterizer.cpp:100-135) ----
constexpr int kSmallSortCap = 2048;
constexpr int kBigSortCap = 16384;
// With ro.rec set, every key's blend record (blend_rec.cuh) is written at the
// key's final position as well (the TMA-staged blend reads them contiguously).
void launch_tile_sort(const uint32_t* offsets, const uint32_t* order, int n_tiles,
                      unsigned long long* keys, cudaStream_t s, RecOut ro = {}, int tiles_x = 1);
void launch_tile_sort_big(const uint32_t* offsets, unsigned long long* keys,
                          const uint32_t* big_list, FrameCounters* cnt, int grid,
                          cudaStream_t s, RecOut ro = {}, int tiles_x = 1);

// ---- blend (rasterizer.cpp:137-165, blend_scalar.cpp:13-55) ----
// Fast-blend kernels (certified-identical): kBlendCpa (default: one
// producer warp, per-lane cp.async into a stage ring completed by the copies),
// kBlendWsp (round 1: two producer warps that cull), kBlendTma (`records` holds
// blend_record_bytes() per pair written by the sort when records_packed, else by a
// pack pass here; each tile's records stream into shared memory with cp.async.bulk),
// kBlendGather4 (TMA tile::gather4 of the n_records slot-indexed 64-byte g32 rows).
enum BlendKernel { kBlendWsp = 0, kBlendTma = 1, kBlendGather4 = 2, kBlendCpa = 3 };
// Banded blend of a synchronous frame: each band's image rows are copied to the host
// while the next band blends (GpuScene::enqueue_pipeline).
constexpr int kMaxBands = 8;
void launch_band_order(const uint32_t* order, int n_tiles, int tiles_x, int band_rows,
                       int n_bands, uint32_t* out, unsigned* tickets, cudaStream_t s);
// k_blend_cpa over the n_order tiles of `order` only (one band); frame_tiles picks the
// ring depth as for the whole frame
void launch_blend_tiles(const uint32_t* offsets, const uint32_t* order, int n_order,
                        int frame_tiles, const unsigned long long* keys, const Gauss64* g64,
                        const Gauss32* g32, int width, int height, int tiles_x, unsigned* ticket,
                        float* image, cudaStream_t s);
void launch_blend(const uint32_t* offsets, const uint32_t* order, const unsigned long long* keys,
                  const Gauss64* g64, const Gauss32* g32, const GaussCol64* col64, int width,
                  int height, int tiles_x, int tiles_y, bool exact, float* image, cudaStream_t s,
                  unsigned* ticket = nullptr, void* records = nullptr, uint64_t n_records = 0,
                  bool records_packed = false, int kernel = kBlendWsp);
uint64_t blend_record_bytes();
int blend_launches();

// Exact blend + per-pair KPC in the reference's 4-lane order (collect_kpc).
void launch_blend_exact_kpc(const uint32_t* offsets, const unsigned long long* keys,
                            const Gauss64* g64, const Gauss32* g32, const GaussCol64* col64,
                            int width, int height, int tiles_x, int tiles_y, float* image,
                            double* kpc, cudaStream_t s);
// Calibration pieces (metrics.cpp:18-57): per-tile GTC, view GTC (NaN when no
// tile has pairs), and the 5-bin kpc redundancy histogram (accumulated).
void launch_view_gtc(const uint32_t* offsets, int n_tiles, const double* kpc, uint64_t n_pairs,
                     double* tile_gtc, double* view_gtc, unsigned long long* bins, cudaStream_t s);

// ---- stage-entry helpers ----
// Reference-order binning of an arbitrary gaussian list: counts, chained scan,
// row-major emission (rasterizer.cpp:75-98).
void launch_bin_reference_order(const GaussEmit* emit, uint64_t n, int tiles_x,
                                unsigned long long* status, FrameCounters* cnt,
                                uint32_t* out_triples /* nullable */, uint64_t cap,
                                int grid, cudaStream_t s);
// Standalone sort_pairs: bucket arbitrary triples by tile, key = depth<<32|input index.
void launch_bucket_triples(const uint32_t* triples, uint64_t n, uint32_t* tile_count,
                           cudaStream_t s);
void launch_scatter_triples(const uint32_t* triples, uint64_t n, uint32_t* cursor,
                            unsigned long long* keys, cudaStream_t s);
void launch_gather_triples(const uint32_t* offsets, int n_tiles, const unsigned long long* keys,
                           const uint32_t* in_triples, uint32_t* out_triples, cudaStream_t s);
// Standalone alpha_blend: sorted triples -> per-tile keys (order kept).
void launch_triples_to_keys(const uint32_t* triples, uint64_t n, unsigned long long* keys,
                            cudaStream_t s);
// BlendList (FP64 SoA) -> blend records.
void launch_pack_blendlist(uint64_t n, const double* mx, const double* my, const double* ca,
                           const double* cb, const double* cc, const double* op,
                           const double* cr, const double* cg, const double* cbl,
                           const double* radius, const float* depth, int tiles_x, int tiles_y,
                           Gauss64* g64, Gauss32* g32, GaussCol64* col64, GaussEmit* emit,
                           cudaStream_t s);
// Collect-mode readback: sorted keys -> (tile, depth, gaussian) triples.
void launch_keys_to_triples(const uint32_t* offsets, int n_tiles, const unsigned long long* keys,
                            const uint32_t* g_of_slot /* nullable */, uint32_t* out_triples,
                            cudaStream_t s);
// Per-gaussian pair counts (bin_to_tiles multiplicity) from emit records.
void launch_gauss_counts(const GaussEmit* emit, const FrameCounters* cnt, uint64_t cap,
                         uint32_t* out, cudaStream_t s);

// zeroes `bytes` (a multiple of 16) with a kernel, not a memset
void launch_zero(void* p, uint64_t bytes, cudaStream_t s);

// ---- scene ingest (scene.cpp:89-165, scene_io.cpp:90-116) ----
// has_child (n bytes, scratch) then the per-node rule masks (9 bits, see
// ingest.cu) and their total; level_begin: n_levels device words.
void launch_validate_nodes(const float* soa, const uint32_t* parent, const uint8_t* leaf,
                           uint8_t* has_child, uint64_t n, const uint64_t* level_begin,
                           int n_levels, uint16_t* mask, unsigned long long* n_bad,
                           cudaStream_t s);
// LDGS v1 payload (after the 20-byte header) -> 14 float SoA arrays + parent + leaf
void launch_deinterleave(const uint8_t* payload, uint64_t n, float* soa, uint32_t* parent,
                         uint8_t* leaf, cudaStream_t s);
// out2[0] = 1 + last non-leaf index (0 if none), out2[1] = bits of max |m|_1 (double)
void launch_tree_extents(const float* soa, const uint8_t* leaf, uint64_t n,
                         unsigned long long* out2, cudaStream_t s);

// ---- image metrics + 8-bit output (metrics.cpp:121-195, image.cpp:12-28) ----
constexpr int kMetricParts = 1184;  // per-CTA partial sums, summed in index order
void launch_rgb8(const float* img, uint64_t n, uint8_t* out, cudaStream_t s);
// *out = sum (double(a[i]) - double(b[i]))^2; partial: kMetricParts doubles
void launch_sq_diff(const float* a, const float* b, uint64_t n, double* partial, double* out,
                    cudaStream_t s);
// *out = sum over all 11x11 windows of the per-window SSIM (metrics.cpp:150-191)
void launch_ssim(const float* a, const float* b, int width, int height, const double* weights,
                 double* partial, double* out, cudaStream_t s);

}  // namespace fgs
