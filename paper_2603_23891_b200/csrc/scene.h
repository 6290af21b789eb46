// scene.h -- device scene (replicated LoD tree) and the per-frame pipeline.
#pragma once

#include <cstdint>
#include <memory>
#include <array>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "host_util.h"
#include "launch.h"

namespace fgs {

void cuda_check(cudaError_t e, const char* what);
#define FGS_CUDA(x) ::fgs::cuda_check((x), #x)

// Owning device allocation (no copy, move-only).
template <class T>
struct DevBuf {
    T* p = nullptr;
    uint64_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(uint64_t count) {
        if (count <= n && p) return;
        release();
        const uint64_t c = count ? count : 1;
        FGS_CUDA(cudaMalloc(&p, c * sizeof(T)));
        n = c;
    }
    uint64_t bytes() const { return n * sizeof(T); }
};

// Makes `device` current for the lifetime of the guard.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int device);
    ~DeviceGuard();
};

// Per-frame scratch sized for one image resolution.
struct ResolutionBuffers {
    int width = 0, height = 0, tiles_x = 0, tiles_y = 0;
    DevBuf<uint32_t> tile_offsets, tile_cursor, big_list, tile_order;
    DevBuf<float> image;
};

// Device staging of a tree before validation and packing: 14 float SoA
// arrays (mean xyz, scale xyz, quat wxyz, opacity, colour rgb), parent, leaf.
struct IngestStage {
    DevBuf<float> soa;
    DevBuf<uint32_t> parent;
    DevBuf<uint8_t> leaf;
};

class GpuScene {
public:
    GpuScene(const lodgs_tree_view& tree, int device);
    // load_scene (scene_io.cpp:213-226) for LDGS v1 binary files, straight to the
    // device: the payload streams through two pinned buffers into device memory,
    // is de-interleaved and validated by kernels.  `timing_ms` (nullable, 3):
    // read+H2D, de-interleave, validate+pack wall times.
    GpuScene(const std::string& ldgs_path, int device, double* timing_ms);
    ~GpuScene();

    void reserve_pairs(uint64_t n);
    uint64_t device_bytes() const;

    // One frame, enqueued only.  Counters for the frame land in host_counters()
    // once the stream reaches the end of the frame.
    void enqueue_frame(const lodgs_camera& cam, const lodgs_render_params& p, float* image_host,
                       bool prefiltered = false);
    // Wait + stats of the last frame.  Throws Error on overflow / non-finite.
    void finish(lodgs_render_stats* stats);
    void render(const lodgs_camera& cam, const lodgs_render_params& p, float* image_host,
                lodgs_render_stats* stats);
    void render_batch(const lodgs_camera* cams, uint64_t n, const lodgs_render_params& p,
                      float* const* images_host, lodgs_render_stats* stats);

    // stage entry points
    uint64_t filter(const lodgs_camera& cam, double tau_r, std::vector<uint32_t>& out);
    // filter_serial (filter.cpp:60-113): level-wise, one kernel + barrier per
    // level; passes = barriers = levels with an active node.  level_ms
    // (nullable, n_levels entries) receives each level's device time.
    uint64_t filter_serial(const lodgs_camera& cam, double tau_r, std::vector<uint32_t>& out,
                           int32_t* passes, double* level_ms);
    int n_levels() const { return int(level_begin_.size()); }
    void mark(const lodgs_camera& cam, uint64_t begin, uint64_t end, double tau_r, uint8_t* vis,
              uint8_t* qpass, double* radius);
    uint64_t prepare(const lodgs_camera& cam, const uint32_t* selected, uint64_t n_sel,
                     int kind, double tau, lodgs_blend_list* out);

    // readbacks of the last frame
    void read_image(float* out);
    const float* image_device() const { return res_.image.p; }
    // floats of the current frame's image (buffers may be larger after a
    // resolution change: DevBuf only ever grows)
    uint64_t image_floats() const { return uint64_t(res_.width) * res_.height * 3; }
    uint64_t read_selected(uint32_t* out, uint64_t cap);
    uint64_t read_pairs(lodgs_tile_pair* out, uint64_t cap);
    uint64_t read_gaussians(lodgs_blend_list* out, uint64_t cap);
    void read_counts(uint32_t* per_gaussian, uint64_t cap_g, uint32_t* per_tile, uint64_t cap_t);
    void take_totals(uint64_t* frames, uint64_t* sum_sel, uint64_t* sum_pairs,
                     uint64_t* sum_sort_bytes = nullptr);
    void take_totals_own(uint64_t* frames, uint64_t* sum_sel, uint64_t* sum_pairs,
                         uint64_t* sum_sort_bytes);
    uint64_t read_kpc(double* out, uint64_t cap);
    void calibrate(const lodgs_camera* views, uint32_t n_views, double lambda_g, double tau_r,
                   lodgs_calibration* out, double* per_view);

    // 8-bit RGB of the current image (save_ppm quantisation, image.cpp:19-22)
    void read_image_rgb8(uint8_t* out);
    // Snapshot the current image as the on-device comparison reference, and
    // psnr / ssim (metrics.cpp:121-192) of the current image against it.
    void set_reference_image();
    void compare_reference(double* psnr, double* ssim);

    // Frames in flight (1 to kMaxInflight, default 4): render_async and
    // render_batch rotate frames over this context and chained twin contexts
    // (own stream and per-frame buffers, same device tree), forked from the
    // control stream; join() makes the control stream wait for all of them.
    // stream() is the control stream.
    void set_inflight(int n);
    void set_sh(int degree, const float* sh_rest, uint64_t n_nodes);
    uint32_t sh_launches() const { return tree_.sh_k > 0 ? 1u : 0u; }
    void enqueue_async(const lodgs_camera& cam, const lodgs_render_params& p, float* image_host);
    // n frames over the in-flight contexts, the filter shared by each group of up to
    // kMaxViews consecutive frames (launch_filter_views); else as enqueue_async
    void enqueue_views_async(const lodgs_camera* cams, uint64_t n, const lodgs_render_params& p,
                             float* const* images_host = nullptr);
    void join();
    void sync_async(lodgs_render_stats* stats);

    void profile(bool enable);
    uint64_t profile_read(double stage_ms[6]);

    cudaStream_t stream() const { return ctl_ ? ctl_ : stream_; }
    int device() const { return device_; }
    uint64_t n_nodes() const { return tree_.n; }

    float shrink_factor() const { return shrink_factor_; }
    const std::vector<uint64_t>& level_begin() const { return level_begin_; }

private:
    struct TwinTag {};
    GpuScene(const GpuScene& owner, TwinTag);
    void alloc_frame_buffers(uint64_t pairs);
    void init_device(int device);
    void init_control();
    void ingest(uint64_t n, const std::vector<uint64_t>& level_begin, bool per_node,
                std::vector<std::string>& msgs, uint64_t nv, IngestStage& st);
    void ensure_resolution(int w, int h);
    void build_readback_maps();
    void clear_frame_state();
    void enqueue_pipeline(const Geom& g, const lodgs_render_params& p, int w, int h, bool timing,
                          bool prefiltered = false);
    void check_frame(const lodgs_camera& cam, const lodgs_render_params& p) const;

    int device_;
    cudaStream_t stream_ = nullptr;
    DevTree tree_;
    std::vector<uint64_t> level_begin_;  // scene.hpp:53 level_begin(l), host copy
    float shrink_factor_ = 0.5f;
    // frames in flight
#ifndef FGS_INFLIGHT_DEFAULT
#define FGS_INFLIGHT_DEFAULT 4
#endif
    static constexpr int kMaxInflight = 12;
    int inflight_ = FGS_INFLIGHT_DEFAULT;
    GpuScene* context(int i);
    void make_contexts(int n);
    std::unique_ptr<GpuScene> twin_;
    cudaStream_t ctl_ = nullptr;
    cudaEvent_t fork_ev_ = nullptr, join_ev_[kMaxInflight] = {};
    cudaEvent_t view_ev_ = nullptr;  // this context's last enqueued work (multi-view groups)
    uint64_t async_frames_ = 0;
    GpuScene* last_frame_ = nullptr;
    DevBuf<unsigned> level_flag_;        // serial filter: level had an active node
    bool last_serial_ = false;
    // tree storage
    DevBuf<float4> geo_;       // (mean, max scale) per node
    DevBuf<float4> iscale_;    // internal region: (scales, leaf flag)
    DevBuf<float4> iquat_;     // internal region: quaternion
    DevBuf<uint32_t> parent_;
    DevBuf<SplatRec> splat_;
    DevBuf<float4> sh_;        // SH rest coefficients (set_sh), tree_.sh_stride per node
    // frame storage
    DevBuf<uint32_t> cand_bits_, qint_bits_, selected_;
    DevBuf<uint2> tile_lists_;       // K3 -> K4 per-CTA (tile, count) entries (<= kHistMaxTiles)
    DevBuf<uint32_t> tile_list_len_;
    DevBuf<Gauss64> g64_;
    DevBuf<Gauss32> g32_;
    DevBuf<GaussEmit> emit_;
    DevBuf<GaussCol64> col64_;
    DevBuf<unsigned long long> keys_;
    DevBuf<unsigned char> blend_rec_;  // per pair, K6a -> K6b (blend_record_bytes() each)
    DevBuf<double> kpc_;         // per sorted pair (collect_kpc frames only)
    bool last_kpc_ = false;
    DevBuf<float> ref_image_;    // comparison reference (set_reference_image)
    int ref_w_ = 0, ref_h_ = 0;
    DevBuf<uint8_t> rgb8_;
    DevBuf<double> metric_partial_;  // kMetricParts + 2
    DevBuf<double> tile_gtc_;    // calibration scratch: per tile, + view result
    DevBuf<unsigned long long> kpc_bins_;
    // readback-only: slot <-> BlendList index maps and compacted records
    DevBuf<uint32_t> g_of_slot_, slot_of_g_;
    DevBuf<Gauss64> rb_g64_;
    DevBuf<Gauss32> rb_g32_;
    DevBuf<GaussEmit> rb_emit_;
    bool maps_valid_ = false;
    uint64_t pair_cap_ = 0;
    // zeroed every frame: [FrameCounters | select status | prep status | tile counts]
    DevBuf<unsigned char> zero_;
    uint64_t zero_bytes_ = 0;
    FrameCounters* d_counters_ = nullptr;
    unsigned long long* d_status_select_ = nullptr;
    unsigned long long* d_status_prep_ = nullptr;
    uint32_t* d_tile_count_ = nullptr;
    uint64_t tile_count_cap_ = 0;
    DevBuf<RunTotals> totals_;
    ResolutionBuffers res_;
    FrameCounters* h_counters_ = nullptr;  // pinned
    cudaEvent_t ev_[6] = {};
    bool last_timing_ = false;
    bool last_keep_ = false;
    bool last_exact_ = false;
    // pipelined batches: second image buffer, copy stream, per-frame counters
    float* image_target_ = nullptr;  // blend output override (nullptr: res_.image)
    // banded blend + copy of a frame with a host image (enqueue_frame -> enqueue_pipeline):
    // each band's rows go to band_host_ on copy_stream_ while the next band blends
    float* band_host_ = nullptr;
    bool band_copied_ = false;
    uint32_t band_launches_ = 0;  // extra launches of the last banded frame (stats)
    DevBuf<uint32_t> band_order_;
    DevBuf<unsigned> band_ticket_;
    cudaEvent_t band_ev_[kMaxBands] = {}, band_done_ = nullptr;
    void ensure_copy_stream();
// render_batch's image ring: the blend of frame i waits for the D2H copy of frame
// i - kBatchBufs; a deeper ring absorbs the jitter between the (faster) compute and the
// PCIe-bound copies (e2e f32 frames/s, cfg 3: 3 / 4 / 6 buffers 2,033-2,047 / 2,082-2,103 /
// 2,129; the link alone moves 56.4 GB/s = 2,265 frames/s)
#ifndef FGS_BATCH_BUFS
#define FGS_BATCH_BUFS 6
#endif
    static constexpr int kBatchBufs = FGS_BATCH_BUFS;  // render_batch image ring
    DevBuf<float> image2_[kBatchBufs - 1];
    DevBuf<uint8_t> rgb8b_[kBatchBufs];  // render_batch with LODGS_RENDER_OUTPUT_RGB8
    cudaStream_t copy_stream_ = nullptr;
    cudaEvent_t frame_done_[kBatchBufs] = {}, copy_done_[kBatchBufs] = {};
    FrameCounters* h_batch_counters_ = nullptr;
    DevBuf<FrameCounters> frame_log_;      // device-side per-frame counters of a batch
    FrameCounters* log_target_ = nullptr;  // enqueue_pipeline: where k_tile_offsets logs
    uint64_t h_batch_cap_ = 0;
    bool profiling_ = false;
    std::vector<std::array<cudaEvent_t, 6>> prof_events_;
    size_t prof_used_ = 0;
    int persistent_grid_ = 148 * 4;
    int sm_count_ = 148;
};

// Stateless per-device context for the stage functions that take no scene
// (bin_to_tiles / sort_pairs / alpha_blend).
void stage_bin_to_tiles(const lodgs_blend_list& list, int width, int height,
                        lodgs_tile_pair* out, uint64_t cap, uint64_t* n_pairs);
void stage_sort_pairs(lodgs_tile_pair* pairs, uint64_t n);
// psnr / ssim of two host images (W*H*3 floats) on the current device;
// ssim may be null.  Throws ValidationError as metrics.cpp:122-149.
void stage_image_metrics(const float* a, const float* b, int width, int height, double* psnr,
                         double* ssim);
// metrics on device images (any device pointers on the current device)
void device_image_metrics(const float* a, const float* b, int width, int height, double* psnr,
                          double* ssim, double* partial, cudaStream_t s);
void stage_alpha_blend(const lodgs_tile_pair* sorted, uint64_t n, const lodgs_blend_list& list,
                       int width, int height, uint32_t flags, float* image);

}  // namespace fgs
