// scene.cpp -- device scene and per-frame pipeline orchestration.
//
// The reference render() (rasterizer.cpp:167-213) validates the tree, then
// runs filter -> prepare -> bin -> sort -> blend with a worker-pool join after
// every pass.  Here the tree is validated and uploaded once; a frame is ten
// stream-ordered kernels with every data-dependent size (N_sel, N_g, N_P)
// kept on the device, so a frame needs no host round trip until its stats
// are read.
#include "scene.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

// fast-blend kernel of a frame without a LODGS_RENDER_BLEND_* flag (experiment builds
// override it)
#ifndef FGS_DEFAULT_BLEND
#define FGS_DEFAULT_BLEND kBlendCpa
#endif

namespace fgs {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(LODGS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

DeviceGuard::DeviceGuard(int device) {
    FGS_CUDA(cudaGetDevice(&prev));
    if (prev != device) FGS_CUDA(cudaSetDevice(device));
}
DeviceGuard::~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
}

void launch_pack_tree(const float* soa, const float* extra, const uint8_t* leaf, uint64_t n,
                      uint64_t leaf_begin, float4* geo, float4* iscale, float4* iquat,
                      SplatRec* splat, cudaStream_t s);
void launch_update_totals(const FrameCounters* cnt, const uint32_t* offsets, int n_tiles,
                          RunTotals* totals, cudaStream_t s);
void launch_max_tile(const uint32_t* triples, uint64_t n, unsigned int* out, cudaStream_t s);

namespace {
uint64_t align256(uint64_t b) { return (b + 255) / 256 * 256; }
}  // namespace

void GpuScene::init_control() {
    // the control stream (timing events, fork/join of in-flight frames)
    FGS_CUDA(cudaStreamCreateWithFlags(&ctl_, cudaStreamNonBlocking));
    FGS_CUDA(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming));
    for (auto& e : join_ev_) FGS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

void GpuScene::init_device(int device) {
    int count = 0;
    FGS_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
        throw Error(LODGS_ERR_CUDA, "device " + std::to_string(device) + " not present");
    DeviceGuard dg(device_);
    FGS_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    FGS_CUDA(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, device_));
    persistent_grid_ = sm_count_ * 4;
    for (auto& e : ev_) FGS_CUDA(cudaEventCreate(&e));
    FGS_CUDA(cudaMallocHost(&h_counters_, sizeof(FrameCounters)));
    std::memset(h_counters_, 0, sizeof(FrameCounters));
}

GpuScene::GpuScene(const lodgs_tree_view& tree, int device) : device_(device) {
    // tree-level rules on the host (cheap), per-node rules on the device
    std::vector<std::string> msgs;
    uint64_t nv = 0;
    const bool per_node = validate_tree_header(tree, msgs, nv);
    if (!per_node && nv) throw Error(LODGS_ERR_VALIDATION, join_violations("invalid tree", msgs, nv));
    init_device(device);
    DeviceGuard dg(device_);
    init_control();
    const uint64_t n = tree.n_nodes;
    IngestStage st;
    st.soa.alloc(14 * n);
    st.parent.alloc(n);
    st.leaf.alloc(n);
    const float* src[14] = {tree.mean_x, tree.mean_y, tree.mean_z, tree.scale_x,
                            tree.scale_y, tree.scale_z, tree.quat_w, tree.quat_x,
                            tree.quat_y, tree.quat_z, tree.opacity, tree.color_r,
                            tree.color_g, tree.color_b};
    if (n) {
        for (int k = 0; k < 14; ++k)
            FGS_CUDA(cudaMemcpyAsync(st.soa.p + k * n, src[k], n * 4, cudaMemcpyHostToDevice,
                                     stream_));
        FGS_CUDA(cudaMemcpyAsync(st.parent.p, tree.parent, n * 4, cudaMemcpyHostToDevice, stream_));
        FGS_CUDA(cudaMemcpyAsync(st.leaf.p, tree.leaf, n, cudaMemcpyHostToDevice, stream_));
    }
    std::vector<uint64_t> lb;
    for (uint32_t l = 0; l < tree.n_levels; ++l) lb.push_back(tree.level_offsets[l]);
    shrink_factor_ = tree.shrink_factor;
    ingest(n, lb, per_node, msgs, nv, st);
    // the other in-flight contexts exist from the start, so no allocation ever
    // lands inside a caller's timed loop of render_async frames
    make_contexts(inflight_);
}

namespace {
struct FileCloser {
    FILE* f;
    ~FileCloser() {
        if (f) std::fclose(f);
    }
};
}  // namespace

GpuScene::GpuScene(const std::string& path, int device, double* timing_ms) : device_(device) {
    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw Error(LODGS_ERR_IO, "cannot open for read: " + path);
    FileCloser closer{f};
    // scene_io.cpp:216-222: a leading '{' (after whitespace) is a JSON scene
    int head = std::fgetc(f);
    while (head == ' ' || head == '\t' || head == '\r' || head == '\n') head = std::fgetc(f);
    if (head == EOF) throw Error(LODGS_ERR_VALIDATION, "bad magic");
    if (head == '{')
        throw Error(LODGS_ERR_VALIDATION,
                    "JSON scene: the device loader reads LDGS v1 binary; load JSON on the host "
                    "(scene_io.cpp:153-198) and create the scene from arrays");
    std::fseek(f, 0, SEEK_SET);
    std::fseek(f, 0, SEEK_END);
    const uint64_t fsize = uint64_t(std::ftell(f));
    std::fseek(f, 0, SEEK_SET);
    // scene_io.cpp:90-116 header, with the reference's messages
    auto rd = [&](void* p, size_t nb, const char* what) {
        if (std::fread(p, 1, nb, f) != nb)
            throw Error(LODGS_ERR_VALIDATION, std::string("truncated scene file reading ") + what);
    };
    char magic[4];
    rd(magic, 4, "magic");
    if (std::memcmp(magic, "LDGS", 4) != 0) throw Error(LODGS_ERR_VALIDATION, "bad magic");
    uint32_t version = 0, n32 = 0, nl = 0;
    float shrink = 0.f;
    rd(&version, 4, "version");
    if (version != 1)
        throw Error(LODGS_ERR_VALIDATION, "unsupported version " + std::to_string(version));
    rd(&n32, 4, "node count");
    rd(&nl, 4, "level count");
    rd(&shrink, 4, "shrink factor");
    const uint64_t n = n32;
    const struct { const char* what; uint64_t bytes; } sections[] = {
        {"means", 12 * n}, {"scales", 12 * n}, {"quaternions", 16 * n}, {"opacity", 4 * n},
        {"colors", 12 * n}, {"parents", 4 * n}, {"leaf flags", n}, {"level offsets", 4ull * nl}};
    uint64_t off = 20;
    for (const auto& sec : sections) {
        if (fsize < off + sec.bytes)
            throw Error(LODGS_ERR_VALIDATION,
                        std::string("truncated scene file reading ") + sec.what);
        off += sec.bytes;
    }
    const uint64_t payload = 61 * n;  // 14 floats + parent + leaf per node
    std::vector<uint32_t> offs(nl);
    std::fseek(f, long(20 + payload), SEEK_SET);
    if (nl) rd(offs.data(), 4ull * nl, "level offsets");
    std::fseek(f, 20, SEEK_SET);
    // tree-level rules (scene.cpp:93-116); per-node rules run on the device
    static const float dummy = 0.f;
    static const uint32_t dummy_u = 0;
    static const uint8_t dummy_b = 0;
    lodgs_tree_view v{};
    v.n_nodes = n;
    v.mean_x = v.mean_y = v.mean_z = v.scale_x = v.scale_y = v.scale_z = &dummy;
    v.quat_w = v.quat_x = v.quat_y = v.quat_z = v.opacity = &dummy;
    v.color_r = v.color_g = v.color_b = &dummy;
    v.parent = &dummy_u;
    v.leaf = &dummy_b;
    v.level_offsets = offs.data();
    v.n_levels = nl;
    v.shrink_factor = shrink;
    std::vector<std::string> msgs;
    uint64_t nv = 0;
    const bool per_node = validate_tree_header(v, msgs, nv);
    if (!per_node && nv) throw Error(LODGS_ERR_VALIDATION, join_violations("invalid tree", msgs, nv));
    init_device(device);
    DeviceGuard dg(device_);
    init_control();
    // payload -> device through two pinned chunks (read of chunk k+1 overlaps the copy of k)
    DevBuf<uint8_t> dpay;
    dpay.alloc(payload);
    constexpr uint64_t kChunk = 32ull << 20;
    uint8_t* pin[2] = {nullptr, nullptr};
    cudaEvent_t done[2];
    for (int k = 0; k < 2; ++k) {
        FGS_CUDA(cudaMallocHost(&pin[k], kChunk));
        FGS_CUDA(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
    }
    try {
        uint64_t pos = 0;
        int k = 0;
        bool used[2] = {false, false};
        while (pos < payload) {
            const uint64_t nb = std::min<uint64_t>(kChunk, payload - pos);
            if (used[k]) FGS_CUDA(cudaEventSynchronize(done[k]));
            if (std::fread(pin[k], 1, nb, f) != nb)
                throw Error(LODGS_ERR_IO, "read failed: " + path);
            FGS_CUDA(cudaMemcpyAsync(dpay.p + pos, pin[k], nb, cudaMemcpyHostToDevice, stream_));
            FGS_CUDA(cudaEventRecord(done[k], stream_));
            used[k] = true;
            pos += nb;
            k ^= 1;
        }
        FGS_CUDA(cudaStreamSynchronize(stream_));
    } catch (...) {
        for (int k = 0; k < 2; ++k) {
            cudaFreeHost(pin[k]);
            cudaEventDestroy(done[k]);
        }
        throw;
    }
    for (int k = 0; k < 2; ++k) {
        cudaFreeHost(pin[k]);
        cudaEventDestroy(done[k]);
    }
    const auto t1 = clock::now();
    IngestStage st;
    st.soa.alloc(14 * n);
    st.parent.alloc(n);
    st.leaf.alloc(n);
    launch_deinterleave(dpay.p, n, st.soa.p, st.parent.p, st.leaf.p, stream_);
    FGS_CUDA(cudaGetLastError());
    FGS_CUDA(cudaStreamSynchronize(stream_));
    dpay.release();
    const auto t2 = clock::now();
    std::vector<uint64_t> lb(offs.begin(), offs.end());
    shrink_factor_ = shrink;
    ingest(n, lb, per_node, msgs, nv, st);
    // the other in-flight contexts exist from the start, so no allocation ever
    // lands inside a caller's timed loop of render_async frames
    make_contexts(inflight_);
    const auto t3 = clock::now();
    if (timing_ms) {
        auto ms = [](clock::time_point a, clock::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        timing_ms[0] = ms(t0, t1);
        timing_ms[1] = ms(t1, t2);
        timing_ms[2] = ms(t2, t3);
    }
}

void GpuScene::ingest(uint64_t n, const std::vector<uint64_t>& level_begin, bool per_node,
                      std::vector<std::string>& msgs, uint64_t nv, IngestStage& st) {
    level_begin_ = level_begin;
    if (per_node && n) {
        // scene.cpp:118-162 on the device: one pass for has_child, one for the rules
        DevBuf<uint8_t> has_child;
        has_child.alloc(n);
        DevBuf<uint16_t> mask;
        mask.alloc(n);
        DevBuf<uint64_t> dlb;
        dlb.alloc(level_begin.size());
        DevBuf<unsigned long long> bad;
        bad.alloc(1);
        FGS_CUDA(cudaMemcpyAsync(dlb.p, level_begin.data(), level_begin.size() * 8,
                                 cudaMemcpyHostToDevice, stream_));
        FGS_CUDA(cudaMemsetAsync(bad.p, 0, 8, stream_));
        launch_validate_nodes(st.soa.p, st.parent.p, st.leaf.p, has_child.p, n, dlb.p,
                              int(level_begin.size()), mask.p, bad.p, stream_);
        FGS_CUDA(cudaGetLastError());
        unsigned long long h_bad = 0;
        FGS_CUDA(cudaMemcpyAsync(&h_bad, bad.p, 8, cudaMemcpyDeviceToHost, stream_));
        FGS_CUDA(cudaStreamSynchronize(stream_));
        if (h_bad) {  // error path: the first messages in (node, rule) order
            std::vector<uint16_t> hm(n);
            FGS_CUDA(cudaMemcpy(hm.data(), mask.p, n * 2, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < n && msgs.size() < 9; ++i)
                for (int k = 0; k < 9 && msgs.size() < 9; ++k)
                    if ((hm[i] >> k) & 1u)
                        msgs.push_back("node " + std::to_string(i) + ": " + node_rule_name(k));
            nv += h_bad;
        }
    }
    if (nv) throw Error(LODGS_ERR_VALIDATION, join_violations("invalid tree", msgs, nv));

    // per-node arrays padded to 256 nodes: the filter's vector loads never run
    // past an allocation
    const uint64_t np = (n + 255) / 256 * 256;
    tree_.n = n;
    DevBuf<unsigned long long> ext;
    ext.alloc(2);
    launch_tree_extents(st.soa.p, st.leaf.p, n, ext.p, stream_);
    unsigned long long h_ext[2] = {0, 0};
    FGS_CUDA(cudaMemcpyAsync(h_ext, ext.p, 16, cudaMemcpyDeviceToHost, stream_));
    FGS_CUDA(cudaStreamSynchronize(stream_));
    // first index of the all-leaf suffix, rounded up to 1024 nodes
    tree_.leaf_begin = std::min<uint64_t>(n, (h_ext[0] + 1023) / 1024 * 1024);
    double max_l1 = 0.0;
    std::memcpy(&max_l1, &h_ext[1], 8);
    tree_.max_l1 = max_l1 * (1.0 + 0x1p-40);
    const uint64_t nb = tree_.leaf_begin;
    geo_.alloc(np);
    FGS_CUDA(cudaMemsetAsync(geo_.p, 0, geo_.bytes(), stream_));
    iscale_.alloc(nb);
    iquat_.alloc(nb);
    splat_.alloc(n);
    launch_pack_tree(st.soa.p, st.soa.p + 6 * n, st.leaf.p, n, nb, geo_.p, iscale_.p, iquat_.p,
                     splat_.p, stream_);
    parent_.alloc(np);
    FGS_CUDA(cudaMemsetAsync(parent_.p, 0xFF, np * 4, stream_));
    if (n) FGS_CUDA(cudaMemcpyAsync(parent_.p, st.parent.p, n * 4, cudaMemcpyDeviceToDevice, stream_));
    FGS_CUDA(cudaStreamSynchronize(stream_));
    tree_.geo = geo_.p;
    tree_.iscale = iscale_.p;
    tree_.iquat = iquat_.p;
    tree_.parent = parent_.p;
    tree_.splat = splat_.p;
    alloc_frame_buffers(std::max<uint64_t>(4 * n, 1u << 16));
}

void GpuScene::alloc_frame_buffers(uint64_t pairs) {
    const uint64_t n = tree_.n;
    cand_bits_.alloc(bit_words(n));
    qint_bits_.alloc(bit_words(n));
    selected_.alloc(n);
    g64_.alloc(n);
    g32_.alloc(n);
    emit_.alloc(n);
    reserve_pairs(pairs);  // grown on overflow
    totals_.alloc(1);
    FGS_CUDA(cudaMemsetAsync(totals_.p, 0, sizeof(RunTotals), stream_));
    FGS_CUDA(cudaStreamSynchronize(stream_));
}

// A second frame context over the same device tree (frames in flight): its own
// stream, counters and per-frame buffers; the tree storage stays the owner's.
GpuScene::GpuScene(const GpuScene& owner, TwinTag) : device_(owner.device_) {
    init_device(device_);
    DeviceGuard dg(device_);
    tree_ = owner.tree_;
    level_begin_ = owner.level_begin_;
    shrink_factor_ = owner.shrink_factor_;
    alloc_frame_buffers(owner.pair_cap_);
}

// Frame contexts in flight: this scene (0), twin_ (1), twin_->twin_ (2).  Each
// twin owns its stream, counters and per-frame buffers over the shared tree;
// the per-context operations (reserve, resolution, totals, memory) recurse.
GpuScene* GpuScene::context(int i) {
    GpuScene* c = this;
    for (; c && i > 0; --i) c = c->twin_.get();
    return c;
}

void GpuScene::make_contexts(int n) {
    GpuScene* c = this;
    for (int i = 1; i < n; ++i) {
        if (!c->twin_) c->twin_.reset(new GpuScene(*c, TwinTag{}));
        c = c->twin_.get();
    }
}

// SH degree 1..3 coefficients (lodgs_gpu_scene_set_sh): packed per node into whole
// float4s, shared by every frame context.  Frames already in flight finish first.
void GpuScene::set_sh(int degree, const float* host, uint64_t n) {
    if (degree < 0 || degree > 3) throw Error(LODGS_ERR_VALIDATION, "sh: degree is 0 to 3");
    DeviceGuard dg(device_);
    for (int i = 0; i < kMaxInflight; ++i)
        if (GpuScene* c = context(i)) FGS_CUDA(cudaStreamSynchronize(c->stream_));
    int k = 0, stride = 0;
    if (degree > 0) {
        if (n != tree_.n) throw Error(LODGS_ERR_VALIDATION, "sh: one row of coefficients per node");
        if (!host) throw Error(LODGS_ERR_VALIDATION, "sh: null coefficients");
        k = (degree + 1) * (degree + 1) - 1;
        stride = (3 * k + 3) / 4;
        std::vector<float> pack(size_t(n) * size_t(stride) * 4, 0.0f);
        for (uint64_t i = 0; i < n; ++i)
            for (int j = 0; j < 3 * k; ++j) {
                const float v = host[i * uint64_t(3 * k) + uint64_t(j)];
                if (!std::isfinite(v))
                    throw Error(LODGS_ERR_VALIDATION,
                                "sh: coefficient of node " + std::to_string(i) + " is not finite");
                pack[i * uint64_t(stride) * 4 + uint64_t(j)] = v;
            }
        sh_.release();
        sh_.alloc(n * uint64_t(stride));
        FGS_CUDA(cudaMemcpy(sh_.p, pack.data(), pack.size() * sizeof(float), cudaMemcpyHostToDevice));
    } else {
        sh_.release();
    }
    for (int i = 0; i < kMaxInflight; ++i)
        if (GpuScene* c = context(i)) {
            c->tree_.sh = degree > 0 ? sh_.p : nullptr;
            c->tree_.sh_k = k;
            c->tree_.sh_stride = stride;
        }
}

void GpuScene::set_inflight(int n) {
    if (n < 1 || n > kMaxInflight)
        throw Error(LODGS_ERR_VALIDATION, "frames in flight: 1 to 12");
    join();
    inflight_ = n;
    make_contexts(n);
}

void GpuScene::enqueue_views_async(const lodgs_camera* cams, uint64_t n,
                                   const lodgs_render_params& p, float* const* images_host) {
    DeviceGuard dg(device_);
    constexpr uint32_t kPerFrameOnly = LODGS_RENDER_STAGE_TIMING | LODGS_RENDER_FILTER_SERIAL |
                                       LODGS_RENDER_COLLECT_KPC | LODGS_RENDER_KEEP_PAIRS;
    bool same_res = true;
    for (uint64_t i = 0; i < n; ++i) {
        check_frame(cams[i], p);
        same_res = same_res && cams[i].width == cams[0].width && cams[i].height == cams[0].height;
    }
    if (n == 0) return;
    // groups of V views alternate between two disjoint sets of V contexts, so a group's
    // filter waits only for the frames of the group before last, and overlaps the
    // previous group's pipelines (one set would drain the GPU between groups)
    const int V = std::min(kMaxViews, inflight_ / 2);
    if (V < 2 || profiling_ || !ctl_ || (p.flags & kPerFrameOnly) || !same_res) {
        for (uint64_t i = 0; i < n; ++i)
            enqueue_async(cams[i], p, images_host ? images_host[i] : nullptr);
        return;
    }
    make_contexts(inflight_);
    ensure_resolution(int(cams[0].width), int(cams[0].height));  // every context follows
    const int nsets = inflight_ / V;  // >= 2 disjoint sets of V contexts, used in turn
    for (uint64_t base = 0; base < n; base += uint64_t(V)) {
        const int nv = int(std::min<uint64_t>(uint64_t(V), n - base));
        GpuScene* ctx[kMaxViews] = {};
        for (int j = 0; j < nv; ++j) {
            ctx[j] = context(int((async_frames_ + uint64_t(j)) % uint64_t(nsets * V)));
            if (!ctx[j]->view_ev_)
                FGS_CUDA(cudaEventCreateWithFlags(&ctx[j]->view_ev_, cudaEventDisableTiming));
        }
        async_frames_ += uint64_t(V);  // the next group starts on the other context set
        // the group's filter runs on its first context's stream, after the control
        // stream's work and after every member context's previous frame
        cudaStream_t fs = ctx[0]->stream_;
        FGS_CUDA(cudaEventRecord(fork_ev_, ctl_));
        FGS_CUDA(cudaStreamWaitEvent(fs, fork_ev_, 0));
        ViewSet vs;
        vs.n = nv;
        for (int j = 0; j < nv; ++j) {
            if (j > 0) {
                FGS_CUDA(cudaEventRecord(ctx[j]->view_ev_, ctx[j]->stream_));
                FGS_CUDA(cudaStreamWaitEvent(fs, ctx[j]->view_ev_, 0));
            }
            launch_zero(ctx[j]->zero_.p, ctx[j]->zero_bytes_, fs);
            vs.g[j] = camera_geom(cams[base + uint64_t(j)]);
            vs.cand[j] = ctx[j]->cand_bits_.p;
            vs.qint[j] = ctx[j]->qint_bits_.p;
            vs.tile_count[j] = reinterpret_cast<uint32_t*>(ctx[j]->d_status_select_);
            vs.selected[j] = ctx[j]->selected_.p;
            vs.cnt[j] = ctx[j]->d_counters_;
        }
        launch_filter_views(vs, tree_, p.tau_r, fs);
        FGS_CUDA(cudaGetLastError());
        FGS_CUDA(cudaEventRecord(ctx[0]->view_ev_, fs));
        for (int j = 0; j < nv; ++j) {
            if (j > 0) FGS_CUDA(cudaStreamWaitEvent(ctx[j]->stream_, ctx[0]->view_ev_, 0));
            ctx[j]->enqueue_frame(cams[base + uint64_t(j)], p,
                                  images_host ? images_host[base + uint64_t(j)] : nullptr,
                                  /*prefiltered=*/true);
        }
        last_frame_ = ctx[nv - 1];
    }
}

void GpuScene::join() {
    if (!ctl_) return;
    DeviceGuard dg(device_);
    for (int i = 0; i < kMaxInflight; ++i) {
        GpuScene* c = context(i);
        if (!c) continue;
        FGS_CUDA(cudaEventRecord(join_ev_[i], c->stream_));
        FGS_CUDA(cudaStreamWaitEvent(ctl_, join_ev_[i], 0));
    }
}

void GpuScene::enqueue_async(const lodgs_camera& cam, const lodgs_render_params& p,
                             float* image_host) {
    DeviceGuard dg(device_);
    if (inflight_ < 2 || profiling_ || !ctl_) {
        if (ctl_) {  // still ordered after the control stream's events
            FGS_CUDA(cudaEventRecord(fork_ev_, ctl_));
            FGS_CUDA(cudaStreamWaitEvent(stream_, fork_ev_, 0));
        }
        enqueue_frame(cam, p, image_host);
        last_frame_ = this;
        return;
    }
    make_contexts(inflight_);
    GpuScene* tgt = context(int(async_frames_++ % uint64_t(inflight_)));
    // fork from the control stream: the frame orders after the caller's events
    // there (e.g. a timing start), not after the other contexts' frames
    FGS_CUDA(cudaEventRecord(fork_ev_, ctl_));
    FGS_CUDA(cudaStreamWaitEvent(tgt->stream_, fork_ev_, 0));
    tgt->enqueue_frame(cam, p, image_host);
    last_frame_ = tgt;
}

void GpuScene::sync_async(lodgs_render_stats* stats) {
    DeviceGuard dg(device_);
    join();
    if (ctl_) FGS_CUDA(cudaStreamSynchronize(ctl_));
    (last_frame_ ? last_frame_ : this)->finish(stats);
}

GpuScene::~GpuScene() {
    cudaSetDevice(device_);
    if (twin_) {
        cudaStreamSynchronize(twin_->stream_);
        twin_.reset();
    }
    if (ctl_) {
        cudaStreamSynchronize(ctl_);
        cudaStreamDestroy(ctl_);
        cudaEventDestroy(fork_ev_);
        for (auto& e : join_ev_) cudaEventDestroy(e);
    }
    if (stream_) cudaStreamSynchronize(stream_);
    if (view_ev_) cudaEventDestroy(view_ev_);
    for (auto& e : ev_)
        if (e) cudaEventDestroy(e);
    for (auto& a : prof_events_)
        for (auto& e : a) cudaEventDestroy(e);
    if (h_counters_) cudaFreeHost(h_counters_);
    if (h_batch_counters_) cudaFreeHost(h_batch_counters_);
    if (copy_stream_) {
        cudaStreamSynchronize(copy_stream_);
        cudaStreamDestroy(copy_stream_);
        for (int k = 0; k < kBatchBufs; ++k) {
            cudaEventDestroy(frame_done_[k]);
            cudaEventDestroy(copy_done_[k]);
        }
    }
    if (band_done_) {
        for (auto& e : band_ev_) cudaEventDestroy(e);
        cudaEventDestroy(band_done_);
    }
    if (stream_) cudaStreamDestroy(stream_);
}

void GpuScene::reserve_pairs(uint64_t n) {
    DeviceGuard dg(device_);
    if (twin_) twin_->reserve_pairs(n);
    if (n > 0xFFFFFFF0ull) n = 0xFFFFFFF0ull;
    if (n <= pair_cap_) return;
    if (stream_) FGS_CUDA(cudaStreamSynchronize(stream_));
    keys_.release();
    keys_.alloc(n);
    if (blend_rec_.p) {  // the TMA blend's per-pair records, once that kernel has been used
        blend_rec_.release();
        blend_rec_.alloc(n * blend_record_bytes());
    }
    pair_cap_ = n;
}

uint64_t GpuScene::device_bytes() const {
    return (twin_ ? twin_->device_bytes() : 0) + geo_.bytes() + iscale_.bytes() + iquat_.bytes() +
           parent_.bytes() + splat_.bytes() + sh_.bytes() +
           cand_bits_.bytes() + qint_bits_.bytes() + selected_.bytes() + g64_.bytes() +
           tile_lists_.bytes() + tile_list_len_.bytes() +
           g32_.bytes() + emit_.bytes() + col64_.bytes() + keys_.bytes() + blend_rec_.bytes() +
           zero_.bytes() +
           res_.tile_offsets.bytes() + res_.tile_cursor.bytes() + res_.big_list.bytes() +
           res_.image.bytes();
}

void GpuScene::ensure_resolution(int w, int h) {
    // the other in-flight contexts follow (recursively), so their first frame at
    // a new resolution never allocates inside a caller's stream of async frames
    if (twin_) twin_->ensure_resolution(w, h);
    if (w == res_.width && h == res_.height && zero_.p) return;
    FGS_CUDA(cudaStreamSynchronize(stream_));
    res_.width = w;
    res_.height = h;
    res_.tiles_x = (w + kTile - 1) / kTile;
    res_.tiles_y = (h + kTile - 1) / kTile;
    const uint64_t n_tiles = uint64_t(res_.tiles_x) * res_.tiles_y;
    if (res_.tiles_x > 32767 || res_.tiles_y > 32767)
        throw Error(LODGS_ERR_VALIDATION, "image too large for 16-bit tile coordinates");
    res_.tile_offsets.alloc(n_tiles + 1);
    res_.tile_cursor.alloc(n_tiles + 1);
    res_.big_list.alloc(n_tiles + 1);
    res_.tile_order.alloc(n_tiles + 1);
    res_.image.alloc(uint64_t(w) * h * 3);
    // render_batch's second image and 8-bit staging: sized with the resolution so
    // no batch call allocates (a first cudaMalloc there cost tens of ms)
    for (auto& im : image2_) im.alloc(uint64_t(w) * h * 3);
    if (n_tiles <= uint64_t(kHistMaxTiles)) {
        tile_lists_.alloc(uint64_t(persistent_grid_) * n_tiles);
        tile_list_len_.alloc(uint64_t(persistent_grid_));
    }
    for (auto& b8 : rgb8b_) b8.alloc(uint64_t(w) * h * 3);
    rgb8_.alloc(uint64_t(w) * h * 3);
    const uint64_t b_cnt = align256(sizeof(FrameCounters));
    const uint64_t b_sel = align256(uint64_t(filter_status_entries(tree_.n)) * 4);
    const uint64_t b_prep = align256((tree_.n / kPrepBlock + 2) * 8);
    const uint64_t b_tiles = align256((n_tiles + 1) * 4);
    zero_bytes_ = b_cnt + b_sel + b_prep + b_tiles;
    zero_.release();
    zero_.alloc(zero_bytes_);
    d_counters_ = reinterpret_cast<FrameCounters*>(zero_.p);
    d_status_select_ = reinterpret_cast<unsigned long long*>(zero_.p + b_cnt);
    d_status_prep_ = reinterpret_cast<unsigned long long*>(zero_.p + b_cnt + b_sel);
    d_tile_count_ = reinterpret_cast<uint32_t*>(zero_.p + b_cnt + b_sel + b_prep);
    tile_count_cap_ = n_tiles;
    FGS_CUDA(cudaMemsetAsync(zero_.p, 0, zero_bytes_, stream_));
    FGS_CUDA(cudaMemsetAsync(res_.tile_offsets.p, 0, res_.tile_offsets.bytes(), stream_));
}

void GpuScene::clear_frame_state() {
    launch_zero(zero_.p, zero_bytes_, stream_);  // zero_bytes_ is 256-aligned
}

void GpuScene::enqueue_pipeline(const Geom& g, const lodgs_render_params& p, int w, int h,
                                bool timing, bool prefiltered) {
    (void)w;
    (void)h;
    const int n_tiles = res_.tiles_x * res_.tiles_y;
    const bool kpc = (p.flags & LODGS_RENDER_COLLECT_KPC) != 0;
    const bool exact = kpc || (p.flags & LODGS_RENDER_EXACT_BLEND) != 0;
    if (exact && col64_.n < tree_.n) col64_.alloc(tree_.n);
    if (kpc && kpc_.n < pair_cap_) kpc_.alloc(pair_cap_);
    last_kpc_ = kpc;
    cudaEvent_t* pe = nullptr;
    if (profiling_) {
        if (prof_used_ == prof_events_.size()) {
            std::array<cudaEvent_t, 6> a;
            for (auto& e : a) FGS_CUDA(cudaEventCreate(&e));
            prof_events_.push_back(a);
        }
        pe = prof_events_[prof_used_++].data();
    }
    if (!prefiltered) clear_frame_state();
    if (timing) FGS_CUDA(cudaEventRecord(ev_[0], stream_));
    if (pe) FGS_CUDA(cudaEventRecord(pe[0], stream_));
    if (prefiltered) {
        // selected list and counters already in place (enqueue_views_async)
    } else if (p.flags & LODGS_RENDER_FILTER_SERIAL) {
        level_flag_.alloc(uint64_t(n_levels()) + 1);
        FGS_CUDA(cudaMemsetAsync(level_flag_.p, 0, level_flag_.bytes(), stream_));
        launch_filter_serial(g, tree_, p.tau_r, level_begin_.data(), n_levels(), cand_bits_.p,
                             qint_bits_.p, reinterpret_cast<uint32_t*>(d_status_select_),
                             level_flag_.p, selected_.p, d_counters_, nullptr, stream_,
                             timing ? &d_counters_->clock : nullptr);
        if (pe) FGS_CUDA(cudaEventRecord(pe[1], stream_));
    } else {
        launch_filter(g, tree_, p.tau_r, cand_bits_.p, qint_bits_.p,
                      reinterpret_cast<uint32_t*>(d_status_select_), selected_.p, d_counters_,
                      stream_, pe ? pe[1] : nullptr, timing ? &d_counters_->clock : nullptr);
    }
    last_serial_ = (p.flags & LODGS_RENDER_FILTER_SERIAL) != 0;
    if (timing) FGS_CUDA(cudaEventRecord(ev_[1], stream_));
    if (pe) FGS_CUDA(cudaEventRecord(pe[2], stream_));
    const bool lists = n_tiles <= kHistMaxTiles && tile_lists_.p;
    PrepOut out{g64_.p, g32_.p, emit_.p, exact ? col64_.p : nullptr, d_tile_count_,
                lists ? tile_lists_.p : nullptr, lists ? tile_list_len_.p : nullptr};
    launch_preprocess(g, tree_, selected_.p, tree_.n, p.shrink_kind, p.tau, res_.tiles_x,
                      res_.tiles_y, out, d_counters_, persistent_grid_, stream_,
                      /*known_visible=*/true);
    launch_sh_colour(g, tree_, emit_.p, g32_.p, out.col64, d_counters_, persistent_grid_, stream_);
    launch_tile_offsets(d_tile_count_, n_tiles, res_.tile_offsets.p, res_.tile_cursor.p,
                        res_.big_list.p, res_.tile_order.p, d_counters_, pair_cap_, stream_,
                        totals_.p, log_target_);
    launch_emit_keys(emit_.p, d_counters_, res_.tiles_x, n_tiles, res_.tile_cursor.p, keys_.p,
                     persistent_grid_, stream_, lists ? tile_lists_.p : nullptr,
                     lists ? tile_list_len_.p : nullptr);
    maps_valid_ = false;
    if (timing) FGS_CUDA(cudaEventRecord(ev_[2], stream_));
    if (pe) FGS_CUDA(cudaEventRecord(pe[3], stream_));
    // fast-blend kernel (LODGS_RENDER_BLEND_*); the TMA one reads per-pair records that
    // the sort writes next to each key
    const int bk = (p.flags & LODGS_RENDER_BLEND_GATHER4) ? kBlendGather4
                   : (p.flags & LODGS_RENDER_BLEND_TMA)   ? kBlendTma
                   : (p.flags & LODGS_RENDER_BLEND_CPA)   ? kBlendCpa
                   : (p.flags & LODGS_RENDER_BLEND_WSP)   ? kBlendWsp
                                                           : FGS_DEFAULT_BLEND;
    if (bk == kBlendTma && !exact && blend_rec_.n < pair_cap_ * blend_record_bytes())
        blend_rec_.alloc(pair_cap_ * blend_record_bytes());
    const RecOut ro{(bk == kBlendTma && !exact) ? reinterpret_cast<BlendRec*>(blend_rec_.p)
                                                 : nullptr,
                    g64_.p, g32_.p};
    launch_tile_sort(res_.tile_offsets.p, res_.tile_order.p, n_tiles, keys_.p, stream_, ro,
                     res_.tiles_x);
    launch_tile_sort_big(res_.tile_offsets.p, keys_.p, res_.big_list.p, d_counters_,
                         sm_count_, stream_, ro, res_.tiles_x);
    if (timing) FGS_CUDA(cudaEventRecord(ev_[3], stream_));
    if (pe) FGS_CUDA(cudaEventRecord(pe[4], stream_));
    float* img_out = image_target_ ? image_target_ : res_.image.p;
    if (p.flags & LODGS_RENDER_COLLECT_KPC) {
        launch_blend_exact_kpc(res_.tile_offsets.p, keys_.p, g64_.p, g32_.p, col64_.p, res_.width,
                               res_.height, res_.tiles_x, res_.tiles_y, img_out, kpc_.p, stream_);
    } else if (band_host_ && bk == kBlendCpa && !exact && !image_target_ && res_.tiles_y >= 2) {
        // synchronous frame with a host image: blend kSyncBands horizontal bands (each
        // in heavy-first tile order) and copy each band's rows to the host while the
        // next one blends -- the D2H of the f32 image (~440 us at 1080p) then overlaps
        // the blend instead of following it
#ifndef FGS_SYNC_BANDS
#define FGS_SYNC_BANDS 4
#endif
        constexpr int kSyncBands = FGS_SYNC_BANDS;
        static_assert(kSyncBands <= kMaxBands, "band tickets");
        const int band_rows = (res_.tiles_y + kSyncBands - 1) / kSyncBands;
        const int nbands = (res_.tiles_y + band_rows - 1) / band_rows;
        band_order_.alloc(uint64_t(n_tiles));
        band_ticket_.alloc(kMaxBands);
        ensure_copy_stream();
        launch_band_order(res_.tile_order.p, n_tiles, res_.tiles_x, band_rows, nbands,
                          band_order_.p, band_ticket_.p, stream_);
        const uint64_t row_floats = uint64_t(res_.width) * 3;
        for (int b = 0; b < nbands; ++b) {
            const int r0 = b * band_rows, r1 = std::min(res_.tiles_y, r0 + band_rows);
            launch_blend_tiles(res_.tile_offsets.p, band_order_.p + uint64_t(r0) * res_.tiles_x,
                               (r1 - r0) * res_.tiles_x, n_tiles, keys_.p, g64_.p, g32_.p,
                               res_.width, res_.height, res_.tiles_x, band_ticket_.p + b, img_out,
                               stream_);
            FGS_CUDA(cudaEventRecord(band_ev_[b], stream_));
            FGS_CUDA(cudaStreamWaitEvent(copy_stream_, band_ev_[b], 0));
            const uint64_t y0 = uint64_t(r0) * kTile;
            const uint64_t y1 = std::min<uint64_t>(uint64_t(res_.height), uint64_t(r1) * kTile);
            FGS_CUDA(cudaMemcpyAsync(band_host_ + y0 * row_floats, img_out + y0 * row_floats,
                                     (y1 - y0) * row_floats * sizeof(float),
                                     cudaMemcpyDeviceToHost, copy_stream_));
        }
        FGS_CUDA(cudaEventRecord(band_done_, copy_stream_));
        band_copied_ = true;  // the stream joins the copies after the blend's timing events
        band_launches_ = uint32_t(nbands);  // nbands blends + k_band_order for one blend
    } else {
        launch_blend(res_.tile_offsets.p, res_.tile_order.p, keys_.p, g64_.p, g32_.p, col64_.p,
                     res_.width, res_.height, res_.tiles_x, res_.tiles_y, exact, img_out, stream_,
                     &d_counters_->blend_ticket, blend_rec_.p, g32_.n, ro.rec != nullptr, bk);
    }
    if (timing) FGS_CUDA(cudaEventRecord(ev_[4], stream_));
    if (pe) FGS_CUDA(cudaEventRecord(pe[5], stream_));
    if (band_copied_) FGS_CUDA(cudaStreamWaitEvent(stream_, band_done_, 0));
    FGS_CUDA(cudaGetLastError());
}

void GpuScene::check_frame(const lodgs_camera& cam, const lodgs_render_params& p) const {
    const auto cv = validate_camera(cam);
    if (!cv.empty()) throw Error(LODGS_ERR_VALIDATION, join_violations("invalid camera", cv, cv.size()));
    if (!(p.tau_r > 0)) throw Error(LODGS_ERR_VALIDATION, "filter config: tau_r > 0");
    if (p.shrink_kind < 0 || p.shrink_kind > 2)
        throw Error(LODGS_ERR_VALIDATION, "shrink mode: unknown kind");
    if (p.shrink_kind != LODGS_SHRINK_THREE_SIGMA && !(p.tau > 0.0 && p.tau < 1.0))
        throw Error(LODGS_ERR_VALIDATION,
                    "render: shrink tau in (0,1); adaptive needs calibration first");
}

// prefiltered: the frame's filter already ran (enqueue_views_async) and left its
// selected list and counters in this context's buffers
void GpuScene::enqueue_frame(const lodgs_camera& cam, const lodgs_render_params& p,
                             float* image_host, bool prefiltered) {
    DeviceGuard dg(device_);
    check_frame(cam, p);
    if (!prefiltered) ensure_resolution(int(cam.width), int(cam.height));
    const Geom g = camera_geom(cam);
    last_timing_ = (p.flags & LODGS_RENDER_STAGE_TIMING) != 0;
    last_keep_ = (p.flags & LODGS_RENDER_KEEP_PAIRS) != 0;
    last_exact_ = (p.flags & LODGS_RENDER_EXACT_BLEND) != 0;
    // banded blend + copy only into pinned (page-locked / registered) host memory: a D2H
    // copy into pageable memory blocks the host thread until it has landed, so the bands
    // would serialise (and the stage timers would count the copies); not with stage timing
    band_host_ = nullptr;
    if (image_host && !(p.flags & LODGS_RENDER_OUTPUT_RGB8) && !last_timing_) {
        cudaPointerAttributes attr{};
        if (cudaPointerGetAttributes(&attr, image_host) == cudaSuccess &&
            attr.type == cudaMemoryTypeHost)
            band_host_ = image_host;
        cudaGetLastError();  // a pageable pointer may leave an error behind on old drivers
    }
    band_copied_ = false;
    band_launches_ = 0;
    enqueue_pipeline(g, p, int(cam.width), int(cam.height), last_timing_, prefiltered);
    band_host_ = nullptr;
    FGS_CUDA(cudaMemcpyAsync(h_counters_, d_counters_, sizeof(FrameCounters),
                             cudaMemcpyDeviceToHost, stream_));
    if (image_host && !band_copied_) {
        if (p.flags & LODGS_RENDER_OUTPUT_RGB8) {
            // save_ppm bytes (image.cpp:19-22): the host buffer is W*H*3 bytes
            rgb8_.alloc(image_floats());
            launch_rgb8(res_.image.p, image_floats(), rgb8_.p, stream_);
            FGS_CUDA(cudaMemcpyAsync(image_host, rgb8_.p, image_floats(), cudaMemcpyDeviceToHost,
                                     stream_));
        } else {
            FGS_CUDA(cudaMemcpyAsync(image_host, res_.image.p, image_floats() * sizeof(float),
                                     cudaMemcpyDeviceToHost, stream_));
        }
    }
}

void GpuScene::ensure_copy_stream() {
    if (!copy_stream_) {
        FGS_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
        for (int k = 0; k < kBatchBufs; ++k) {
            FGS_CUDA(cudaEventCreateWithFlags(&frame_done_[k], cudaEventDisableTiming));
            FGS_CUDA(cudaEventCreateWithFlags(&copy_done_[k], cudaEventDisableTiming));
        }
    }
    if (!band_done_) {
        for (auto& e : band_ev_) FGS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        FGS_CUDA(cudaEventCreateWithFlags(&band_done_, cudaEventDisableTiming));
    }
}

void GpuScene::finish(lodgs_render_stats* stats) {
    DeviceGuard dg(device_);
    FGS_CUDA(cudaStreamSynchronize(stream_));
    const FrameCounters c = *h_counters_;
    if (c.overflow) {
        reserve_pairs(std::max<uint64_t>(pair_cap_ * 2, c.n_pairs + c.n_pairs / 4 + 1024));
        throw Error(LODGS_ERR_INTERNAL, "overflow: pair buffer grown, re-render the frame");
    }
    if (c.nonfinite) throw Error(LODGS_ERR_VALIDATION, "projection produced non-finite values");
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->n_selected = c.n_selected;
        stats->n_gaussians = c.n_gaussians;
        stats->n_pairs = c.n_pairs;
        stats->filter_passes = last_serial_ ? int32_t(c.serial_passes) : 2;
        stats->filter_barriers = stats->filter_passes;
        stats->big_tiles = c.big_tiles;
        stats->kernel_launches =
            (last_serial_ ? uint32_t(kLaunchesPerFrame + blend_launches() + n_levels() + filter_launches(tree_.n) - 3 + sh_launches()) : kLaunchesPerFrame + blend_launches() + filter_launches(tree_.n) + sh_launches()) +
            band_launches_;
        if (last_timing_) {
            float ms = 0;
            FGS_CUDA(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
            // filter.cpp:95-96 / :144-145 split the filter into compute (T_calcu) and
            // synchronisation (T_synch).  On the device the passes are kernels and the
            // barriers are the kernel boundaries: T_calcu = the sum over the filter's
            // kernels of first-CTA-start .. last-CTA-end (%globaltimer), T_synch = the
            // rest of the filter's event-timed span (drain, launch and memset gaps).
            double busy = 0.0;
            for (int k = 0; k < kFilterClocks; ++k) {
                const unsigned long long t0 = ~c.clock.t0n[k], t1 = c.clock.t1[k];
                if (c.clock.t1[k] && t1 > t0) busy += double(t1 - t0) * 1e-6;
            }
            busy = std::min(busy, double(ms));
            stats->t_calc_ms = busy;
            stats->t_sync_ms = double(ms) - busy;
            FGS_CUDA(cudaEventElapsedTime(&ms, ev_[1], ev_[2]));
            stats->t_prepr_ms = ms;
            FGS_CUDA(cudaEventElapsedTime(&ms, ev_[2], ev_[3]));
            stats->t_sort_ms = ms;
            FGS_CUDA(cudaEventElapsedTime(&ms, ev_[3], ev_[4]));
            stats->t_alpha_ms = ms;
        }
    }
}

void GpuScene::render(const lodgs_camera& cam, const lodgs_render_params& p, float* image_host,
                      lodgs_render_stats* stats) {
    last_frame_ = this;
    for (int attempt = 0;; ++attempt) {
        enqueue_frame(cam, p, image_host);
        try {
            finish(stats);
            return;
        } catch (const Error& e) {
            if (e.code != LODGS_ERR_INTERNAL || attempt >= 4) throw;
        }
    }
}

void GpuScene::render_batch(const lodgs_camera* cams, uint64_t n, const lodgs_render_params& p,
                            float* const* images_host, lodgs_render_stats* stats) {
    DeviceGuard dg(device_);
    if (n == 0) return;
    for (uint64_t i = 0; i < n; ++i) {
        const auto cv = validate_camera(cams[i]);
        if (!cv.empty())
            throw Error(LODGS_ERR_VALIDATION, join_violations("invalid camera", cv, cv.size()));
        if (cams[i].width != cams[0].width || cams[i].height != cams[0].height)
            throw Error(LODGS_ERR_VALIDATION, "render_batch: all frames share one image size");
    }
    if (!(p.tau_r > 0)) throw Error(LODGS_ERR_VALIDATION, "filter config: tau_r > 0");
    if (p.shrink_kind < 0 || p.shrink_kind > 2)
        throw Error(LODGS_ERR_VALIDATION, "shrink mode: unknown kind");
    if (p.shrink_kind != LODGS_SHRINK_THREE_SIGMA && !(p.tau > 0.0 && p.tau < 1.0))
        throw Error(LODGS_ERR_VALIDATION,
                    "render: shrink tau in (0,1); adaptive needs calibration first");
    ensure_resolution(int(cams[0].width), int(cams[0].height));
    ensure_copy_stream();
    frame_log_.alloc(std::max<uint64_t>(n, 1024));  // one allocation for typical batches
    if (h_batch_cap_ < n) {  // pinned, grown geometrically (cudaMallocHost is slow)
        const uint64_t cap = std::max<uint64_t>(n, std::max<uint64_t>(1024, 2 * h_batch_cap_));
        if (h_batch_counters_) FGS_CUDA(cudaFreeHost(h_batch_counters_));
        FGS_CUDA(cudaMallocHost(&h_batch_counters_, cap * sizeof(FrameCounters)));
        h_batch_cap_ = cap;
    }
    const bool rgb8 = (p.flags & LODGS_RENDER_OUTPUT_RGB8) != 0;
    const uint64_t img_bytes = image_floats() * sizeof(float);
    const uint64_t out_bytes = rgb8 ? image_floats() : img_bytes;
    float* bufs[kBatchBufs];
    bufs[0] = res_.image.p;
    for (int k = 1; k < kBatchBufs; ++k) bufs[k] = image2_[k - 1].p;
    last_timing_ = false;
    last_keep_ = false;
    last_exact_ = (p.flags & LODGS_RENDER_EXACT_BLEND) != 0;
    // frames rotate over the in-flight contexts like render_async (the image
    // ring, the copy stream and the counter log stay this scene's); every
    // context first orders after the work already on this scene's stream
    const int nctx = profiling_ ? 1 : inflight_;
    make_contexts(nctx);
    if (nctx > 1) {
        FGS_CUDA(cudaEventRecord(frame_done_[0], stream_));
        for (int c = 1; c < nctx; ++c)
            FGS_CUDA(cudaStreamWaitEvent(context(c)->stream_, frame_done_[0], 0));
    }
    for (uint64_t i = 0; i < n; ++i) {
        const int k = int(i % kBatchBufs);
        GpuScene* c = context(int(i % uint64_t(nctx)));
        // the blend may overwrite bufs[k] only once the copy out of it (frame
        // i - kBatchBufs) is done
        if (i >= uint64_t(kBatchBufs))
            FGS_CUDA(cudaStreamWaitEvent(c->stream_, copy_done_[k], 0));
        c->image_target_ = bufs[k];
        c->log_target_ = frame_log_.p + i;
        c->enqueue_pipeline(camera_geom(cams[i]), p, int(cams[i].width), int(cams[i].height),
                            false);
        c->image_target_ = nullptr;
        c->log_target_ = nullptr;
        if (rgb8) launch_rgb8(bufs[k], image_floats(), rgb8b_[k].p, c->stream_);
        FGS_CUDA(cudaEventRecord(frame_done_[k], c->stream_));
        FGS_CUDA(cudaStreamWaitEvent(copy_stream_, frame_done_[k], 0));
        if (images_host && images_host[i])
            FGS_CUDA(cudaMemcpyAsync(images_host[i],
                                     rgb8 ? static_cast<const void*>(rgb8b_[k].p) : bufs[k],
                                     out_bytes, cudaMemcpyDeviceToHost, copy_stream_));
        FGS_CUDA(cudaEventRecord(copy_done_[k], copy_stream_));
    }
    for (int c = 1; c < nctx; ++c) FGS_CUDA(cudaStreamSynchronize(context(c)->stream_));
    // every frame's counters in one copy, after the last frame
    FGS_CUDA(cudaMemcpyAsync(h_batch_counters_, frame_log_.p, n * sizeof(FrameCounters),
                             cudaMemcpyDeviceToHost, stream_));
    FGS_CUDA(cudaStreamSynchronize(stream_));
    FGS_CUDA(cudaStreamSynchronize(copy_stream_));
    // the last frame's image also lives in res_.image for read_image()
    if (bufs[(n - 1) % kBatchBufs] != res_.image.p)
        FGS_CUDA(cudaMemcpy(res_.image.p, bufs[(n - 1) % kBatchBufs], img_bytes, cudaMemcpyDeviceToDevice));
    *h_counters_ = h_batch_counters_[n - 1];
    last_frame_ = this;  // read_image & co. read this context's res_.image, not a twin's
    for (uint64_t i = 0; i < n; ++i) {
        const FrameCounters& c = h_batch_counters_[i];
        if (c.nonfinite) throw Error(LODGS_ERR_VALIDATION, "projection produced non-finite values");
        if (c.overflow) {  // rare: grow, then redo this frame synchronously
            reserve_pairs(std::max<uint64_t>(pair_cap_ * 2, c.n_pairs + c.n_pairs / 4 + 1024));
            render(cams[i], p, images_host ? images_host[i] : nullptr,
                   stats ? stats + i : nullptr);
            continue;
        }
        if (stats) {
            lodgs_render_stats& s = stats[i];
            std::memset(&s, 0, sizeof s);
            s.n_selected = c.n_selected;
            s.n_gaussians = c.n_gaussians;
            s.n_pairs = c.n_pairs;
            s.filter_passes = last_serial_ ? int32_t(c.serial_passes) : 2;
            s.filter_barriers = s.filter_passes;
            s.big_tiles = c.big_tiles;
            s.kernel_launches = last_serial_ ? uint32_t(kLaunchesPerFrame + blend_launches() + n_levels() + filter_launches(tree_.n) - 3 + sh_launches())
                                             : kLaunchesPerFrame + blend_launches() + filter_launches(tree_.n) + sh_launches();
        }
    }
}

uint64_t GpuScene::filter(const lodgs_camera& cam, double tau_r, std::vector<uint32_t>& out) {
    DeviceGuard dg(device_);
    if (!(tau_r > 0)) throw Error(LODGS_ERR_VALIDATION, "filter config: tau_r > 0");
    ensure_resolution(int(cam.width), int(cam.height));
    const Geom g = camera_geom(cam);
    clear_frame_state();
    launch_filter(g, tree_, tau_r, cand_bits_.p, qint_bits_.p,
                  reinterpret_cast<uint32_t*>(d_status_select_), selected_.p, d_counters_,
                  stream_);
    FGS_CUDA(cudaMemcpyAsync(h_counters_, d_counters_, sizeof(FrameCounters),
                             cudaMemcpyDeviceToHost, stream_));
    FGS_CUDA(cudaStreamSynchronize(stream_));
    const uint64_t ns = h_counters_->n_selected;
    out.resize(ns);
    if (ns)
        FGS_CUDA(cudaMemcpy(out.data(), selected_.p, ns * 4, cudaMemcpyDeviceToHost));
    return ns;
}

void GpuScene::read_image_rgb8(uint8_t* out) {
    DeviceGuard dg(device_);
    if (last_frame_ && last_frame_ != this) {
        join();
        last_frame_->read_image_rgb8(out);
        return;
    }
    const uint64_t n = image_floats();
    rgb8_.alloc(n);
    launch_rgb8(res_.image.p, n, rgb8_.p, stream_);
    FGS_CUDA(cudaGetLastError());
    FGS_CUDA(cudaMemcpyAsync(out, rgb8_.p, n, cudaMemcpyDeviceToHost, stream_));
    FGS_CUDA(cudaStreamSynchronize(stream_));
}

void GpuScene::set_reference_image() {
    DeviceGuard dg(device_);
    if (!res_.image.p) throw Error(LODGS_ERR_VALIDATION, "set_reference_image: no frame rendered");
    ref_image_.alloc(image_floats());
    FGS_CUDA(cudaMemcpyAsync(ref_image_.p, res_.image.p, image_floats() * 4,
                             cudaMemcpyDeviceToDevice, stream_));
    ref_w_ = res_.width;
    ref_h_ = res_.height;
    FGS_CUDA(cudaStreamSynchronize(stream_));
}

void GpuScene::compare_reference(double* psnr, double* ssim) {
    DeviceGuard dg(device_);
    if (!ref_image_.p || ref_w_ != res_.width || ref_h_ != res_.height)
        throw Error(LODGS_ERR_VALIDATION, "psnr: image dimensions differ");
    metric_partial_.alloc(kMetricParts + 2);
    device_image_metrics(res_.image.p, ref_image_.p, res_.width, res_.height, psnr, ssim,
                         metric_partial_.p, stream_);
}

void device_image_metrics(const float* a, const float* b, int width, int height, double* psnr,
                          double* ssim, double* partial, cudaStream_t s) {
    if (ssim && (width < 11 || height < 11))
        throw Error(LODGS_ERR_VALIDATION, "ssim: images smaller than the 11x11 window");
    const uint64_t n = uint64_t(width) * uint64_t(height) * 3;
    double h[2] = {0.0, 0.0};
    if (psnr) launch_sq_diff(a, b, n, partial, partial + kMetricParts, s);
    if (ssim) {
        double w[121];
        ssim_window(w);
        launch_ssim(a, b, width, height, w, partial, partial + kMetricParts + 1, s);
    }
    FGS_CUDA(cudaGetLastError());
    FGS_CUDA(cudaMemcpyAsync(h, partial + kMetricParts, 16, cudaMemcpyDeviceToHost, s));
    FGS_CUDA(cudaStreamSynchronize(s));
    if (psnr) {
        const double mse = h[0] / double(n);
        *psnr = mse == 0.0 ? INFINITY : 10.0 * std::log10(1.0 / mse);
    }
    if (ssim) *ssim = h[1] / (3.0 * double(width - 10) * double(height - 10));
}

uint64_t GpuScene::filter_serial(const lodgs_camera& cam, double tau_r, std::vector<uint32_t>& out,
                                 int32_t* passes, double* level_ms) {
    DeviceGuard dg(device_);
    if (!(tau_r > 0)) throw Error(LODGS_ERR_VALIDATION, "filter config: tau_r > 0");
    ensure_resolution(int(cam.width), int(cam.height));
    const Geom g = camera_geom(cam);
    const int nl = n_levels();
    clear_frame_state();
    DevBuf<unsigned> flags;
    flags.alloc(uint64_t(nl) + 1);
    FGS_CUDA(cudaMemsetAsync(flags.p, 0, flags.bytes(), stream_));
    std::vector<cudaEvent_t> ev;
    if (level_ms) {
        ev.resize(size_t(nl) + 1);
        for (auto& e : ev) FGS_CUDA(cudaEventCreate(&e));
    }
    launch_filter_serial(g, tree_, tau_r, level_begin_.data(), nl, cand_bits_.p, qint_bits_.p,
                         reinterpret_cast<uint32_t*>(d_status_select_), flags.p, selected_.p,
                         d_counters_, level_ms ? ev.data() : nullptr, stream_);
    FGS_CUDA(cudaGetLastError());
    FGS_CUDA(cudaMemcpyAsync(h_counters_, d_counters_, sizeof(FrameCounters),
                             cudaMemcpyDeviceToHost, stream_));
    std::vector<unsigned> hf(size_t(nl) + 1, 0u);
    if (nl) FGS_CUDA(cudaMemcpyAsync(hf.data(), flags.p, size_t(nl) * 4, cudaMemcpyDeviceToHost, stream_));
    FGS_CUDA(cudaStreamSynchronize(stream_));
    if (level_ms) {
        for (int l = 0; l < nl; ++l) {
            float ms = 0.f;
            FGS_CUDA(cudaEventElapsedTime(&ms, ev[size_t(l)], ev[size_t(l) + 1]));
            level_ms[l] = ms;
        }
        for (auto& e : ev) cudaEventDestroy(e);
    }
    int32_t ps = 0;
    for (int l = 0; l < nl; ++l) ps += hf[size_t(l)] ? 1 : 0;
    if (passes) *passes = ps;
    const uint64_t ns = h_counters_->n_selected;
    out.resize(ns);
    if (ns) FGS_CUDA(cudaMemcpy(out.data(), selected_.p, ns * 4, cudaMemcpyDeviceToHost));
    return ns;
}

void GpuScene::mark(const lodgs_camera& cam, uint64_t begin, uint64_t end, double tau_r,
                    uint8_t* vis, uint8_t* qpass, double* radius) {
    DeviceGuard dg(device_);
    if (end > tree_.n || begin > end) throw Error(LODGS_ERR_VALIDATION, "mark: range out of bounds");
    const uint64_t m = end - begin;
    if (m == 0) return;
    const Geom g = camera_geom(cam);
    DevBuf<uint8_t> dv, dq;
    DevBuf<double> dr;
    dv.alloc(m);
    dq.alloc(m);
    if (radius) dr.alloc(m);
    launch_mark_debug(g, tree_, begin, end, tau_r, dv.p, dq.p, radius ? dr.p : nullptr, stream_);
    FGS_CUDA(cudaGetLastError());
    FGS_CUDA(cudaStreamSynchronize(stream_));
    FGS_CUDA(cudaMemcpy(vis + begin, dv.p, m, cudaMemcpyDeviceToHost));
    FGS_CUDA(cudaMemcpy(qpass + begin, dq.p, m, cudaMemcpyDeviceToHost));
    if (radius) FGS_CUDA(cudaMemcpy(radius + begin, dr.p, m * 8, cudaMemcpyDeviceToHost));
}

uint64_t GpuScene::prepare(const lodgs_camera& cam, const uint32_t* selected, uint64_t n_sel,
                           int kind, double tau, lodgs_blend_list* out) {
    DeviceGuard dg(device_);
    if (n_sel > tree_.n) throw Error(LODGS_ERR_VALIDATION, "prepare: more selected than nodes");
    for (uint64_t i = 0; i < n_sel; ++i)
        if (selected[i] >= tree_.n) throw Error(LODGS_ERR_VALIDATION, "prepare: node index out of range");
    ensure_resolution(int(cam.width), int(cam.height));
    const Geom g = camera_geom(cam);
    clear_frame_state();
    if (n_sel) {
        FGS_CUDA(cudaMemcpyAsync(selected_.p, selected, n_sel * 4, cudaMemcpyHostToDevice, stream_));
        FGS_CUDA(cudaMemcpyAsync(&d_counters_->n_selected, &n_sel, 8, cudaMemcpyHostToDevice, stream_));
    }
    PrepOut po{g64_.p, g32_.p, emit_.p, nullptr, d_tile_count_};
    launch_preprocess(g, tree_, selected_.p, n_sel, kind, tau, res_.tiles_x, res_.tiles_y, po,
                      d_counters_, persistent_grid_, stream_);
    launch_sh_colour(g, tree_, emit_.p, g32_.p, nullptr, d_counters_, persistent_grid_, stream_);
    maps_valid_ = false;
    FGS_CUDA(cudaGetLastError());
    FGS_CUDA(cudaMemcpyAsync(h_counters_, d_counters_, sizeof(FrameCounters),
                             cudaMemcpyDeviceToHost, stream_));
    FGS_CUDA(cudaStreamSynchronize(stream_));
    if (h_counters_->nonfinite) throw Error(LODGS_ERR_VALIDATION, "projection produced non-finite values");
    const uint64_t ng = h_counters_->n_gaussians;
    if (ng && kind != LODGS_SHRINK_THREE_SIGMA && !(tau > 0.0 && tau < 1.0))
        throw Error(LODGS_ERR_VALIDATION, "shrink mode: tau in (0,1)");
    return read_gaussians(out, n_sel);
}

void GpuScene::read_image(float* out) {
    DeviceGuard dg(device_);
    if (last_frame_ && last_frame_ != this) {  // the last async frame ran on the twin
        join();
        last_frame_->read_image(out);
        return;
    }
    FGS_CUDA(cudaStreamSynchronize(stream_));
    FGS_CUDA(cudaMemcpy(out, res_.image.p, image_floats() * sizeof(float), cudaMemcpyDeviceToHost));
}

uint64_t GpuScene::read_selected(uint32_t* out, uint64_t cap) {
    DeviceGuard dg(device_);
    FGS_CUDA(cudaStreamSynchronize(stream_));
    const uint64_t ns = h_counters_->n_selected;
    if (out) {
        if (cap < ns) throw Error(LODGS_ERR_VALIDATION, "read_selected: capacity too small");
        if (ns) FGS_CUDA(cudaMemcpy(out, selected_.p, ns * 4, cudaMemcpyDeviceToHost));
    }
    return ns;
}

// Slot -> BlendList index map and BlendList-ordered copies of the records,
// built on demand for parity readbacks (the hot path never needs them).
void GpuScene::build_readback_maps() {
    if (maps_valid_) return;
    const uint64_t ns = h_counters_->n_selected;
    const uint64_t ng = h_counters_->n_gaussians;
    g_of_slot_.alloc(ns);
    slot_of_g_.alloc(ng);
    rb_g64_.alloc(ng);
    rb_g32_.alloc(ng);
    rb_emit_.alloc(ng);
    FGS_CUDA(cudaMemsetAsync(&d_counters_->ticket_prep, 0, sizeof(unsigned), stream_));
    FGS_CUDA(cudaMemsetAsync(d_status_prep_, 0, (ns / 256 + 2) * 8, stream_));
    launch_slot_map(emit_.p, ns, d_status_prep_, d_counters_, g_of_slot_.p, slot_of_g_.p,
                    persistent_grid_, stream_);
    launch_compact_records(slot_of_g_.p, ng, g64_.p, g32_.p, emit_.p, rb_g64_.p, rb_g32_.p,
                           rb_emit_.p, stream_);
    FGS_CUDA(cudaGetLastError());
    FGS_CUDA(cudaStreamSynchronize(stream_));
    maps_valid_ = true;
}

uint64_t GpuScene::read_pairs(lodgs_tile_pair* out, uint64_t cap) {
    DeviceGuard dg(device_);
    FGS_CUDA(cudaStreamSynchronize(stream_));
    const int n_tiles = res_.tiles_x * res_.tiles_y;
    uint32_t np = 0;
    FGS_CUDA(cudaMemcpy(&np, res_.tile_offsets.p + n_tiles, 4, cudaMemcpyDeviceToHost));
    if (!out) return np;
    if (cap < np) throw Error(LODGS_ERR_VALIDATION, "read_pairs: capacity too small");
    if (np == 0) return 0;
    build_readback_maps();
    DevBuf<uint32_t> tri;
    tri.alloc(uint64_t(np) * 3);
    launch_keys_to_triples(res_.tile_offsets.p, n_tiles, keys_.p, g_of_slot_.p, tri.p, stream_);
    FGS_CUDA(cudaGetLastError());
    FGS_CUDA(cudaStreamSynchronize(stream_));
    FGS_CUDA(cudaMemcpy(out, tri.p, uint64_t(np) * 12, cudaMemcpyDeviceToHost));
    return np;
}

uint64_t GpuScene::read_gaussians(lodgs_blend_list* out, uint64_t cap) {
    DeviceGuard dg(device_);
    FGS_CUDA(cudaStreamSynchronize(stream_));
    const uint64_t ng = h_counters_->n_gaussians;
    if (!out) return ng;
    if (cap < ng) throw Error(LODGS_ERR_VALIDATION, "read_gaussians: capacity too small");
    build_readback_maps();
    std::vector<Gauss64> a(ng);
    std::vector<Gauss32> b(ng);
    std::vector<GaussEmit> e(ng);
    if (ng) {
        FGS_CUDA(cudaMemcpy(a.data(), rb_g64_.p, ng * sizeof(Gauss64), cudaMemcpyDeviceToHost));
        FGS_CUDA(cudaMemcpy(b.data(), rb_g32_.p, ng * sizeof(Gauss32), cudaMemcpyDeviceToHost));
        FGS_CUDA(cudaMemcpy(e.data(), rb_emit_.p, ng * sizeof(GaussEmit), cudaMemcpyDeviceToHost));
    }
    out->n = ng;
    for (uint64_t i = 0; i < ng; ++i) {
        out->mean_x[i] = b[i].mx;
        out->mean_y[i] = b[i].my;
        out->conic_a[i] = a[i].ca;
        out->conic_b[i] = a[i].cb;
        out->conic_c[i] = a[i].cc;
        out->opacity[i] = a[i].op;
        // colours are f32 in the tree: exact (with SH, set_sh, the FP64 colour rounded to
        // f32; the exact blend keeps the FP64 one)
        out->col_r[i] = double(b[i].r);
        out->col_g[i] = double(b[i].g);
        out->col_b[i] = double(b[i].b);
        out->radius[i] = b[i].radius;
        std::memcpy(&out->depth[i], &e[i].depth_bits, 4);
        out->node[i] = e[i].node;
    }
    return ng;
}

void GpuScene::read_counts(uint32_t* per_gaussian, uint64_t cap_g, uint32_t* per_tile,
                           uint64_t cap_t) {
    DeviceGuard dg(device_);
    FGS_CUDA(cudaStreamSynchronize(stream_));
    if (per_gaussian) {
        build_readback_maps();
        DevBuf<uint32_t> tmp;
        tmp.alloc(cap_g);
        launch_gauss_counts(rb_emit_.p, d_counters_, cap_g, tmp.p, stream_);
        FGS_CUDA(cudaGetLastError());
        FGS_CUDA(cudaStreamSynchronize(stream_));
        const uint64_t ng = std::min<uint64_t>(h_counters_->n_gaussians, cap_g);
        if (ng) FGS_CUDA(cudaMemcpy(per_gaussian, tmp.p, ng * 4, cudaMemcpyDeviceToHost));
    }
    if (per_tile) {
        const uint64_t nt = std::min<uint64_t>(tile_count_cap_, cap_t);
        if (nt) FGS_CUDA(cudaMemcpy(per_tile, d_tile_count_, nt * 4, cudaMemcpyDeviceToHost));
    }
}

uint64_t GpuScene::read_kpc(double* out, uint64_t cap) {
    DeviceGuard dg(device_);
    FGS_CUDA(cudaStreamSynchronize(stream_));
    if (!last_kpc_) throw Error(LODGS_ERR_VALIDATION, "read_kpc: last frame had no collect_kpc");
    const int n_tiles = res_.tiles_x * res_.tiles_y;
    uint32_t np = 0;
    FGS_CUDA(cudaMemcpy(&np, res_.tile_offsets.p + n_tiles, 4, cudaMemcpyDeviceToHost));
    if (!out) return np;
    if (cap < np) throw Error(LODGS_ERR_VALIDATION, "read_kpc: capacity too small");
    if (np) FGS_CUDA(cudaMemcpy(out, kpc_.p, uint64_t(np) * 8, cudaMemcpyDeviceToHost));
    return np;
}

// metrics.cpp:79-108 (instrumented_render + calibrate + make_report).
void GpuScene::calibrate(const lodgs_camera* views, uint32_t n_views, double lambda_g,
                         double tau_r, lodgs_calibration* out, double* per_view) {
    DeviceGuard dg(device_);
    if (n_views == 0) throw Error(LODGS_ERR_VALIDATION, "calibration: no views");
    if (!(lambda_g > 0.0)) throw Error(LODGS_ERR_VALIDATION, "calibration: lambda_g > 0 required");
    kpc_bins_.alloc(5);
    FGS_CUDA(cudaMemsetAsync(kpc_bins_.p, 0, 5 * sizeof(unsigned long long), stream_));
    std::vector<double> used;
    for (uint32_t v = 0; v < n_views; ++v) {
        const lodgs_render_params p{tau_r, 0.0, LODGS_SHRINK_THREE_SIGMA, LODGS_RENDER_COLLECT_KPC};
        render(views[v], p, nullptr, nullptr);
        const int n_tiles = res_.tiles_x * res_.tiles_y;
        tile_gtc_.alloc(uint64_t(n_tiles) + 1);
        launch_view_gtc(res_.tile_offsets.p, n_tiles, kpc_.p, h_counters_->n_pairs, tile_gtc_.p,
                        tile_gtc_.p + n_tiles, kpc_bins_.p, stream_);
        FGS_CUDA(cudaGetLastError());
        double g = 0.0;
        FGS_CUDA(cudaMemcpyAsync(&g, tile_gtc_.p + n_tiles, 8, cudaMemcpyDeviceToHost, stream_));
        FGS_CUDA(cudaStreamSynchronize(stream_));
        if (!std::isnan(g)) used.push_back(g);
    }
    // make_report (metrics.cpp:59-77), on the host like the reference
    if (used.empty()) throw Error(LODGS_ERR_VALIDATION, "calibration: no view produced any pairs");
    double sum = 0.0;
    for (double g : used) sum += g;
    const double mean = sum / double(used.size());
    if (!(mean > 0.0)) throw Error(LODGS_ERR_VALIDATION, "calibration: zero mean contribution");
    unsigned long long bins[5];
    FGS_CUDA(cudaMemcpy(bins, kpc_bins_.p, sizeof bins, cudaMemcpyDeviceToHost));
    out->tau = lambda_g / mean;
    out->scene_gtc = mean;
    out->lambda_g = lambda_g;
    out->n_views = uint32_t(used.size());
    for (int k = 0; k < 5; ++k) out->histogram[k] = bins[k];
    if (per_view)
        for (size_t i = 0; i < used.size(); ++i) per_view[i] = used[i];
}

void GpuScene::profile(bool enable) {
    DeviceGuard dg(device_);
    FGS_CUDA(cudaStreamSynchronize(stream_));
    if (enable) prof_used_ = 0;
    profiling_ = enable;
}

uint64_t GpuScene::profile_read(double stage_ms[6]) {
    DeviceGuard dg(device_);
    FGS_CUDA(cudaStreamSynchronize(stream_));
    for (int k = 0; k < 6; ++k) stage_ms[k] = 0.0;
    for (size_t f = 0; f < prof_used_; ++f) {
        const auto& e = prof_events_[f];
        float ms = 0;
        for (int k = 0; k < 5; ++k) {
            FGS_CUDA(cudaEventElapsedTime(&ms, e[k], e[k + 1]));
            stage_ms[k] += ms;
        }
        FGS_CUDA(cudaEventElapsedTime(&ms, e[0], e[5]));
        stage_ms[5] += ms;
    }
    return prof_used_;
}

void GpuScene::take_totals(uint64_t* frames, uint64_t* sum_sel, uint64_t* sum_pairs,
                           uint64_t* sum_sort_bytes) {
    DeviceGuard dg(device_);
    if (twin_) {
        uint64_t f = 0, s = 0, p = 0, b = 0;
        twin_->take_totals(&f, &s, &p, &b);  // throws (after growing) on overflow
        uint64_t f0 = 0, s0 = 0, p0 = 0, b0 = 0;
        take_totals_own(&f0, &s0, &p0, &b0);
        if (frames) *frames = f + f0;
        if (sum_sel) *sum_sel = s + s0;
        if (sum_pairs) *sum_pairs = p + p0;
        if (sum_sort_bytes) *sum_sort_bytes = b + b0;
        return;
    }
    take_totals_own(frames, sum_sel, sum_pairs, sum_sort_bytes);
}

void GpuScene::take_totals_own(uint64_t* frames, uint64_t* sum_sel, uint64_t* sum_pairs,
                               uint64_t* sum_sort_bytes) {
    DeviceGuard dg(device_);
    RunTotals t;
    FGS_CUDA(cudaStreamSynchronize(stream_));
    FGS_CUDA(cudaMemcpy(&t, totals_.p, sizeof t, cudaMemcpyDeviceToHost));
    FGS_CUDA(cudaMemset(totals_.p, 0, sizeof t));
    if (frames) *frames = t.frames;
    if (sum_sel) *sum_sel = t.sum_selected;
    if (sum_pairs) *sum_pairs = t.sum_pairs;
    if (sum_sort_bytes) *sum_sort_bytes = t.sum_sort_bytes;
    if (t.pad) {
        reserve_pairs(pair_cap_ * 2);
        throw Error(LODGS_ERR_INTERNAL, "overflow: pair buffer grown, re-render the frames");
    }
}

// ============================================================================
// Stateless stage functions on the current device.
namespace {

struct StageCtx {
    int device = -1;
    cudaStream_t s = nullptr;
    std::mutex mu;
};

StageCtx& stage_ctx() {
    static std::mutex g;
    static std::map<int, std::unique_ptr<StageCtx>> ctxs;
    int dev = 0;
    FGS_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g);
    auto& c = ctxs[dev];
    if (!c) {
        c = std::make_unique<StageCtx>();
        c->device = dev;
        FGS_CUDA(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking));
    }
    return *c;
}

template <class T>
void upload(DevBuf<T>& d, const T* h, uint64_t n, cudaStream_t s) {
    d.alloc(n);
    if (n) FGS_CUDA(cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
}

struct DevList {
    DevBuf<double> f[10];
    DevBuf<float> depth;
    DevBuf<Gauss64> g64;
    DevBuf<Gauss32> g32;
    DevBuf<GaussCol64> col64;
    DevBuf<GaussEmit> emit;
    void load(const lodgs_blend_list& l, int tiles_x, int tiles_y, bool need_col64,
              cudaStream_t s) {
        const double* src[10] = {l.mean_x, l.mean_y, l.conic_a, l.conic_b, l.conic_c,
                                 l.opacity, l.col_r, l.col_g, l.col_b, l.radius};
        for (int k = 0; k < 10; ++k) {
            if (!src[k] && l.n) throw Error(LODGS_ERR_VALIDATION, "blend list: null array");
            upload(f[k], src[k], l.n, s);
        }
        if (!l.depth && l.n) throw Error(LODGS_ERR_VALIDATION, "blend list: null depth");
        upload(depth, l.depth, l.n, s);
        g64.alloc(l.n);
        g32.alloc(l.n);
        emit.alloc(l.n);
        if (need_col64) col64.alloc(l.n);
        launch_pack_blendlist(l.n, f[0].p, f[1].p, f[2].p, f[3].p, f[4].p, f[5].p, f[6].p,
                              f[7].p, f[8].p, f[9].p, depth.p, tiles_x, tiles_y, g64.p, g32.p,
                              need_col64 ? col64.p : nullptr, emit.p, s);
    }
};

}  // namespace

void stage_bin_to_tiles(const lodgs_blend_list& list, int width, int height,
                        lodgs_tile_pair* out, uint64_t cap, uint64_t* n_pairs) {
    if (width < 1 || height < 1) throw Error(LODGS_ERR_VALIDATION, "bin_to_tiles: image size");
    StageCtx& c = stage_ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    DevList dl;
    dl.load(list, tiles_x, tiles_y, false, c.s);
    DevBuf<unsigned char> z;
    const uint64_t b_cnt = align256(sizeof(FrameCounters));
    const uint64_t b_st = align256((list.n / 256 + 2) * 8);
    z.alloc(b_cnt + b_st);
    FGS_CUDA(cudaMemsetAsync(z.p, 0, b_cnt + b_st, c.s));
    auto* cnt = reinterpret_cast<FrameCounters*>(z.p);
    auto* st = reinterpret_cast<unsigned long long*>(z.p + b_cnt);
    DevBuf<uint32_t> tri;
    if (out && cap) tri.alloc(cap * 3);
    launch_bin_reference_order(dl.emit.p, list.n, tiles_x, st, cnt, out ? tri.p : nullptr, cap,
                               296, c.s);
    FGS_CUDA(cudaGetLastError());
    FrameCounters h;
    FGS_CUDA(cudaMemcpyAsync(&h, cnt, sizeof h, cudaMemcpyDeviceToHost, c.s));
    FGS_CUDA(cudaStreamSynchronize(c.s));
    *n_pairs = h.n_pairs;
    if (out) {
        if (cap < h.n_pairs) throw Error(LODGS_ERR_VALIDATION, "bin_to_tiles: capacity too small");
        if (h.n_pairs) FGS_CUDA(cudaMemcpy(out, tri.p, h.n_pairs * 12, cudaMemcpyDeviceToHost));
    }
}

// Buckets by tile (counting digit), then sorts each bucket on
// depth_bits << 32 | input position -- the stable order of rasterizer.cpp:100-135.
void stage_sort_pairs(lodgs_tile_pair* pairs, uint64_t n) {
    if (n < 2) return;
    if (n >= 0xFFFFFFF0ull) throw Error(LODGS_ERR_VALIDATION, "sort_pairs: too many pairs");
    StageCtx& c = stage_ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    DevBuf<uint32_t> in, outb;
    upload(in, reinterpret_cast<const uint32_t*>(pairs), n * 3, c.s);
    outb.alloc(n * 3);
    DevBuf<unsigned int> mx;
    mx.alloc(1);
    FGS_CUDA(cudaMemsetAsync(mx.p, 0, 4, c.s));
    launch_max_tile(in.p, n, mx.p, c.s);
    unsigned int max_tile = 0;
    FGS_CUDA(cudaMemcpyAsync(&max_tile, mx.p, 4, cudaMemcpyDeviceToHost, c.s));
    FGS_CUDA(cudaStreamSynchronize(c.s));
    if (max_tile >= (1u << 26))
        throw Error(LODGS_ERR_VALIDATION, "sort_pairs: tile id >= 2^26 not supported");
    const int n_buckets = int(max_tile) + 1;
    DevBuf<unsigned char> z;
    const uint64_t b_cnt = align256(sizeof(FrameCounters));
    const uint64_t b_tc = align256(uint64_t(n_buckets + 1) * 4);
    z.alloc(b_cnt + b_tc);
    FGS_CUDA(cudaMemsetAsync(z.p, 0, b_cnt + b_tc, c.s));
    auto* cnt = reinterpret_cast<FrameCounters*>(z.p);
    auto* tc = reinterpret_cast<uint32_t*>(z.p + b_cnt);
    DevBuf<uint32_t> off, cur, big, ord;
    off.alloc(n_buckets + 1);
    cur.alloc(n_buckets + 1);
    big.alloc(n_buckets + 1);
    ord.alloc(n_buckets + 1);
    DevBuf<unsigned long long> keys;
    keys.alloc(n);
    launch_bucket_triples(in.p, n, tc, c.s);
    launch_tile_offsets(tc, n_buckets, off.p, cur.p, big.p, ord.p, cnt, n, c.s);
    launch_scatter_triples(in.p, n, cur.p, keys.p, c.s);
    launch_tile_sort(off.p, ord.p, n_buckets, keys.p, c.s);
    int n_sm = 148;
    FGS_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, c.device));
    launch_tile_sort_big(off.p, keys.p, big.p, cnt, n_sm, c.s);
    launch_gather_triples(off.p, n_buckets, keys.p, in.p, outb.p, c.s);
    FGS_CUDA(cudaGetLastError());
    FGS_CUDA(cudaMemcpyAsync(pairs, outb.p, n * 12, cudaMemcpyDeviceToHost, c.s));
    FGS_CUDA(cudaStreamSynchronize(c.s));
}

void stage_image_metrics(const float* a, const float* b, int width, int height, double* psnr,
                         double* ssim) {
    if (width < 1 || height < 1) throw Error(LODGS_ERR_VALIDATION, "psnr: image dimensions");
    StageCtx& c = stage_ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    const uint64_t n = uint64_t(width) * uint64_t(height) * 3;
    DevBuf<float> da, db;
    da.alloc(n);
    db.alloc(n);
    DevBuf<double> part;
    part.alloc(kMetricParts + 2);
    FGS_CUDA(cudaMemcpyAsync(da.p, a, n * 4, cudaMemcpyHostToDevice, c.s));
    FGS_CUDA(cudaMemcpyAsync(db.p, b, n * 4, cudaMemcpyHostToDevice, c.s));
    device_image_metrics(da.p, db.p, width, height, psnr, ssim, part.p, c.s);
}

void stage_alpha_blend(const lodgs_tile_pair* sorted, uint64_t n, const lodgs_blend_list& list,
                       int width, int height, uint32_t flags, float* image) {
    if (width < 1 || height < 1) throw Error(LODGS_ERR_VALIDATION, "alpha_blend: image size");
    StageCtx& c = stage_ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const int n_tiles = tiles_x * tiles_y;
    for (uint64_t i = 0; i < n; ++i) {
        if (sorted[i].tile >= uint32_t(n_tiles))
            throw Error(LODGS_ERR_VALIDATION, "alpha_blend: tile id outside the image");
        if (sorted[i].gaussian >= list.n)
            throw Error(LODGS_ERR_VALIDATION, "alpha_blend: gaussian index out of range");
        if (i && sorted[i].tile < sorted[i - 1].tile)
            throw Error(LODGS_ERR_VALIDATION, "alpha_blend: pairs not sorted by tile");
    }
    const bool exact = (flags & LODGS_RENDER_EXACT_BLEND) != 0;
    DevList dl;
    dl.load(list, tiles_x, tiles_y, exact, c.s);
    DevBuf<uint32_t> tri;
    upload(tri, reinterpret_cast<const uint32_t*>(sorted), n * 3, c.s);
    DevBuf<unsigned char> z;
    const uint64_t b_cnt = align256(sizeof(FrameCounters));
    const uint64_t b_tc = align256(uint64_t(n_tiles + 1) * 4);
    z.alloc(b_cnt + b_tc);
    FGS_CUDA(cudaMemsetAsync(z.p, 0, b_cnt + b_tc, c.s));
    auto* cnt = reinterpret_cast<FrameCounters*>(z.p);
    auto* tc = reinterpret_cast<uint32_t*>(z.p + b_cnt);
    DevBuf<uint32_t> off, cur, big, ord;
    off.alloc(n_tiles + 1);
    cur.alloc(n_tiles + 1);
    big.alloc(n_tiles + 1);
    ord.alloc(n_tiles + 1);
    DevBuf<unsigned long long> keys;
    keys.alloc(n);
    DevBuf<float> img;
    img.alloc(uint64_t(width) * height * 3);
    launch_bucket_triples(tri.p, n, tc, c.s);
    launch_tile_offsets(tc, n_tiles, off.p, cur.p, big.p, ord.p, cnt, n, c.s);
    launch_triples_to_keys(tri.p, n, keys.p, c.s);
    const int bk = (flags & LODGS_RENDER_BLEND_GATHER4) ? kBlendGather4
                   : (flags & LODGS_RENDER_BLEND_TMA)   ? kBlendTma
                   : (flags & LODGS_RENDER_BLEND_CPA)   ? kBlendCpa
                   : (flags & LODGS_RENDER_BLEND_WSP)   ? kBlendWsp
                                                         : FGS_DEFAULT_BLEND;
    DevBuf<unsigned char> rec;
    if (bk == kBlendTma) rec.alloc(n * blend_record_bytes());
    launch_blend(off.p, ord.p, keys.p, dl.g64.p, dl.g32.p, dl.col64.p, width, height, tiles_x,
                 tiles_y, exact, img.p, c.s, &cnt->blend_ticket, rec.p, dl.g32.n, false, bk);
    FGS_CUDA(cudaGetLastError());
    FGS_CUDA(cudaMemcpyAsync(image, img.p, img.n * 4, cudaMemcpyDeviceToHost, c.s));
    FGS_CUDA(cudaStreamSynchronize(c.s));
}

}  // namespace fgs
