// blend.cu -- tile-wise front-to-back alpha blending (K6), reference
// alpha_blend -> blend_scalar (rasterizer.cpp:137-165, blend_scalar.cpp:13-55).
//
// Fast kernel: one 128-thread CTA per 16x8 half tile; warp w owns an 8x4
// pixel block (8*(w&1), 4*(w>>1)) of the half tile, lane l its pixel
// (l&7, l>>3).  Warps never synchronise with each other: each walks the
// tile's sorted pair list 32 splats at a time, every lane tests one splat's
// conservative alpha>=1/255 box (Gauss32::hx/hy) against the warp's block,
// hits are staged in the warp's own shared-memory slice, and one ballot
// gives the warp an ordered work list.  All control flow on the list is
// warp-uniform, so lanes never drift apart.  The four warps of a CTA read
// the same splat records, which therefore come from L1 after the first.
// A sample outside the box has e > ln(255 op) and is skipped by the
// reference too, so culling never changes a pixel.
//
// FP32 per sample, with the reference's FP64 decision recomputed exactly
// (warp vote, rare) whenever the FP32 estimate is within a certified margin
// of the alpha >= 1/255 threshold -- a flipped skip would move a pixel by up
// to 1/255 (SURVEY.md section 7 hard part 6).  The test needs no exp:
//     alpha = min(op exp(power), 0.99) < 1/255  <=>  e > ln(255 op),
//     e = -power = ha dx^2 + cb dx dy + hc dy^2 >= 0.
// With Q = ha dx^2 + hc dy^2 >= |cb dx dy| (positive-definite conic),
// |e32 - e| is a few ulp of Q, well inside margin = (Q + 1) 2^-17.
// Accepted samples blend branch-free: w = alpha T, C += c w, T -= w.
//
// Exact kernel (LODGS_RENDER_EXACT_BLEND): the reference arithmetic in FP64
// with the reference exp_mx (fastexp.hpp:38-50), no FMA: bit-identical pixels.
#include <algorithm>
#include <mutex>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "blend_rec.cuh"
#include "launch.h"
#include "pdl.cuh"

namespace fgs {

// fastexp.hpp:18-50, same constants, same operation order (-fmad=false).
__device__ __forceinline__ double exp_mx(double x) {
    x = std_max(x, -30.0);
    const double t = x * 1.44269504088896338700e+00;
    const double u = t + 6755399441055744.0;
    const double fn = u - 6755399441055744.0;
    const double r1 = x - fn * 6.93147180369123816490e-01;
    const double r = r1 - fn * 1.90821492927058770002e-10;
    double p = 1.0 / 479001600;
    p = p * r + 1.0 / 39916800;
    p = p * r + 1.0 / 3628800;
    p = p * r + 1.0 / 362880;
    p = p * r + 1.0 / 40320;
    p = p * r + 1.0 / 5040;
    p = p * r + 1.0 / 720;
    p = p * r + 1.0 / 120;
    p = p * r + 1.0 / 24;
    p = p * r + 1.0 / 6;
    p = p * r + 1.0 / 2;
    p = p * r + 1.0;
    p = p * r + 1.0;
    const long long n = static_cast<long long>(fn);
    return p * __longlong_as_double((n + 1023) << 52);
}

// blend_scalar.cpp:24-31 for one sample, FP64.
__device__ __forceinline__ double alpha_exact(double mx, double my, double ca, double cb,
                                              double cc, double op, double px, double py) {
    const double dx = px - mx;
    const double dy = py - my;
    const double t1 = (ca * dx) * dx;
    const double t2 = (cc * dy) * dy;
    const double t3 = (cb * dx) * dy;
    const double power = -0.5 * (t1 + t2) - t3;
    return std_min(op * exp_mx(power), kAlphaCap);
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

constexpr int kFastThreads = 128;  // fast kernel: one CTA per 16x8 half tile
constexpr int kFastWarps = kFastThreads / 32;
constexpr int kFastParts = kTile * kTile / kFastThreads;

// A batch's hits, compacted in pair order: 12 floats per hit.
struct WarpStage {
    float4 geo[32];  // block-relative mean x, y, ha, hc   (log2e-scaled conic)
    float4 ct[32];   // cb, ethr, op, r
    float2 gb[32];   // g, b
    uint32_t gid[32];
};

// One sample of the fast path: e (log2 units) from the staged hit, the
// certified skip test, alpha and the branch-free blend; T == 0 marks a
// terminated pixel (every later w is 0).  `unsure` accumulates |d| <= margin:
// the FP32 decision might differ from the reference's FP64 one.
struct PixState {
    float T, cr, cg, cb;
};
#ifndef BLEND_TMUL
#define BLEND_TMUL 0
#endif

__device__ __forceinline__ void sample_fast(const float4 geo, const float4 ct, const float2 gb,
                                            float pxl, float pyl, PixState& p, bool& unsure) {
    const float dx = pxl - geo.x, dy = pyl - geo.y;
    const float Q = __fmaf_rn(geo.z * dx, dx, geo.w * dy * dy);
    const float ev = __fmaf_rn(ct.x * dx, dy, Q);
    const float d = ev - ct.y;
    // certified: |e32 - e| is a few ulp of Q (+ the rounding of ethr)
    const float margin = __fmaf_rn(Q, 7.62939453125e-06f, 1.1007e-05f);  // (Q + log2 e) 2^-17
    unsure = unsure || fabsf(d) <= margin;
    const float ev_take = d < -margin ? ev : INFINITY;  // skipped: 2^-inf = 0
    const float alpha = fminf(ct.z * ex2_approx(-ev_take), 0.99f);
    const float w = alpha * p.T;
    p.cr = __fmaf_rn(ct.w, w, p.cr);
    p.cg = __fmaf_rn(gb.x, w, p.cg);
    p.cb = __fmaf_rn(gb.y, w, p.cb);
#if BLEND_TMUL  // T (1 - alpha): one dependent operation fewer on the T chain
    const float t = p.T * (1.0f - alpha);
#else
    const float t = p.T - w;
#endif
    p.T = t < 1e-4f ? 0.0f : t;
}

__device__ __forceinline__ void blend_sample_fast(const WarpStage& st, int k, float pxl,
                                                  float pyl, PixState& p, bool& unsure) {
    sample_fast(st.geo[k], st.ct[k], st.gb[k], pxl, pyl, p, unsure);
}

// The same sample with the reference's FP64 decision wherever the FP32 one is
// uncertain (used only to re-run a batch in which some lane was unsure).
__device__ __forceinline__ void sample_checked(const float4 geo, const float4 ct, const float2 gb,
                                               uint32_t gid, float pxl, float pyl, double px,
                                               double py, const Gauss64* __restrict__ g64,
                                               const Gauss32* __restrict__ g32, PixState& p) {
    const float dx = pxl - geo.x, dy = pyl - geo.y;
    const float Q = __fmaf_rn(geo.z * dx, dx, geo.w * dy * dy);
    const float ev = __fmaf_rn(ct.x * dx, dy, Q);
    const float d = ev - ct.y;
    const float margin = __fmaf_rn(Q, 7.62939453125e-06f, 1.1007e-05f);
    bool take = d < -margin;
    float alpha = fminf(ct.z * ex2_approx(-ev), 0.99f);
    if (fabsf(d) <= margin && p.T > 0.0f) {
        const Gauss64& G = g64[gid];
        const double2 m = *reinterpret_cast<const double2*>(&g32[gid].mx);
        const double a64 = alpha_exact(m.x, m.y, G.ca, G.cb, G.cc, G.op, px, py);
        take = a64 >= kMinAlpha;
        alpha = float(a64);
    }
    const float w = take ? alpha * p.T : 0.0f;
    p.cr = __fmaf_rn(ct.w, w, p.cr);
    p.cg = __fmaf_rn(gb.x, w, p.cg);
    p.cb = __fmaf_rn(gb.y, w, p.cb);
#if BLEND_TMUL
    const float t = take ? p.T * (1.0f - alpha) : p.T;
#else
    const float t = p.T - w;
#endif
    p.T = t < 1e-4f ? 0.0f : t;
}

__device__ __forceinline__ void blend_sample_checked(const WarpStage& st, int k, float pxl,
                                                     float pyl, double px, double py,
                                                     const Gauss64* __restrict__ g64,
                                                     const Gauss32* __restrict__ g32,
                                                     PixState& p) {
    sample_checked(st.geo[k], st.ct[k], st.gb[k], st.gid[k], pxl, pyl, px, py, g64, g32, p);
}

#ifndef BLEND_PREFETCH2
#define BLEND_PREFETCH2 0
#endif
#ifndef BLEND_MIN_CTAS
#define BLEND_MIN_CTAS 8
#endif
__global__ void __launch_bounds__(kFastThreads, BLEND_MIN_CTAS) k_blend_fast(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ order,
    const unsigned long long* __restrict__ keys, const Gauss64* __restrict__ g64,
    const Gauss32* __restrict__ g32, const int width, const int height, const int tiles_x,
    float* __restrict__ image) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    __shared__ WarpStage stage[kFastWarps];
    // heaviest tiles first (k_tile_offsets' schedule), halves of a tile adjacent
    const int tile = int(order[blockIdx.x / kFastParts]), part = blockIdx.x % kFastParts;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpStage& st = stage[warp];
    // this warp's 8x4 block origin in image pixels
    const int bx = (tile % tiles_x) * kTile + int(warp & 1) * 8;
    const int by = (tile / tiles_x) * kTile + part * 8 + int(warp >> 1) * 4;
    const int x = bx + int(lane & 7), y = by + int(lane >> 3);
    const bool inside = x < width && y < height;
    const uint32_t b = offsets[tile], e = offsets[tile + 1];

    const float pxl = float(lane & 7) + 0.5f, pyl = float(lane >> 3) + 0.5f;
    const double px = double(x) + 0.5, py = double(y) + 0.5;
    PixState pix{inside ? 1.0f : 0.0f, 0.0f, 0.0f, 0.0f};  // T == 0: nothing to do
    if (__all_sync(0xffffffffu, !inside)) return;
    const unsigned lt = (1u << lane) - 1u;

    // Software pipeline over 32-splat batches: keys are fetched two batches
    // ahead and splat records one batch ahead, so the dependent key -> record
    // global loads overlap the blending of the previous batch.
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    struct Rec {
        double2 m;
        float4 q0, col;
        float2 h;
    };
    auto load_key = [&](uint32_t at) -> uint32_t {
        return at + lane < e ? uint32_t(keys[at + lane]) : kNone;
    };
    auto load_rec = [&](uint32_t gi, Rec& r) {
        if (gi != kNone) {
            r.m = *reinterpret_cast<const double2*>(&g32[gi].mx);
            r.q0 = *reinterpret_cast<const float4*>(&g32[gi].ha);
            r.col = *reinterpret_cast<const float4*>(&g32[gi].op);
            r.h = *reinterpret_cast<const float2*>(&g32[gi].hx);
        }
    };
#if BLEND_PREFETCH2
    uint32_t gi_cur = load_key(b), gi_next = load_key(b + 32), gi_n2 = load_key(b + 64);
    Rec cur, nxt, nx2;
    load_rec(gi_cur, cur);
    load_rec(gi_next, nxt);
#else
    uint32_t gi_cur = load_key(b), gi_next = load_key(b + 32);
    Rec cur, nxt;
    load_rec(gi_cur, cur);
#endif
    for (uint32_t base = b; base < e; base += 32) {
        // ---- stage the splats of this batch that touch this warp's block,
        //      compacted in pair order
        bool hit = false;
        float mlx = 0.f, mly = 0.f;
        if (gi_cur != kNone) {
            mlx = float(cur.m.x - double(bx));
            mly = float(cur.m.y - double(by));
            // pixel centres of the block span [0.5, 7.5] x [0.5, 3.5]
            const float2 h = cur.h;
            hit = h.x >= 0.0f && mlx - h.x <= 7.5f && mlx + h.x >= 0.5f && mly - h.y <= 3.5f &&
                  mly + h.y >= 0.5f;
        }
        const unsigned bits = __ballot_sync(0xffffffffu, hit);
        if (hit) {
            const int slot = __popc(bits & lt);
            st.geo[slot] = make_float4(mlx, mly, cur.q0.x, cur.q0.z);
            st.ct[slot] = make_float4(cur.q0.y, cur.q0.w, cur.col.x, cur.col.y);
            st.gb[slot] = make_float2(cur.col.z, cur.col.w);
            st.gid[slot] = gi_cur;
        }
        __syncwarp();
#if BLEND_PREFETCH2
        // ---- prefetch: records two batches ahead, keys three ahead
        const uint32_t gi_after = load_key(base + 96);
        load_rec(gi_n2, nx2);
#else
        // ---- prefetch: records of the next batch, keys of the one after
        const uint32_t gi_after = load_key(base + 64);
        load_rec(gi_next, nxt);
#endif
        // ---- blend them front to back (FP32; re-run exactly if any lane was unsure)
        const int nh = __popc(bits);
        const PixState saved = pix;
        bool unsure = false;
        int k = 0;
        for (; k + 2 <= nh; k += 2) {
            blend_sample_fast(st, k, pxl, pyl, pix, unsure);
            blend_sample_fast(st, k + 1, pxl, pyl, pix, unsure);
        }
        if (k < nh) blend_sample_fast(st, k, pxl, pyl, pix, unsure);
        if (__any_sync(0xffffffffu, unsure)) {  // rare: certified FP64 decisions
            pix = saved;
            for (int j = 0; j < nh; ++j) blend_sample_checked(st, j, pxl, pyl, px, py, g64, g32, pix);
        }
        if (__all_sync(0xffffffffu, pix.T == 0.0f)) break;
        __syncwarp();
#if BLEND_PREFETCH2
        gi_cur = gi_next;
        gi_next = gi_n2;
        gi_n2 = gi_after;
        cur = nxt;
        nxt = nx2;
#else
        gi_cur = gi_next;
        gi_next = gi_after;
        cur = nxt;
#endif
    }
    if (inside) {
        float* o = image + (size_t(y) * width + x) * 3;
        o[0] = pix.cr;
        o[1] = pix.cg;
        o[2] = pix.cb;
    }
}

// ---------------------------------------------------------------------------
// Warp-specialised fast blend: one CTA per 16x16 tile, 8 consumer warps (one
// 8x4 block each) and 1 producer warp.  The producer walks the tile's sorted
// pairs 32 at a time -- keys two batches and records one batch ahead in
// registers -- culls every splat against all 8 blocks at once and writes each
// block's hits, compacted in pair order, into a ring of kWsStages shared-
// memory stages; mbarriers hand stages over (full: 32 producer lanes, empty:
// 8 x 32 consumer lanes).  Each record is loaded and culled once per tile
// instead of once per warp, and the ring depth hides the gather latency.
// Consumers run the same per-sample code as k_blend_fast.
#ifndef WS_STAGES
#define WS_STAGES 5
#endif
constexpr int kWsStages = WS_STAGES;
constexpr int kWsConsumers = 8;
#ifndef WS_PRODUCERS
#define WS_PRODUCERS 2
#endif
#ifndef WS_NOSTOP
#define WS_NOSTOP 0  // timing experiment: no early stop of saturated tiles
#endif
#ifndef WS_NOCONSUME
#define WS_NOCONSUME 0  // timing experiment: producers only
#endif
#ifndef WS_HINT
#define WS_HINT 0  // suspend-time hint (ns) of the mbarrier waits (0: none)
#endif
#ifndef WS_SLEEP
#define WS_SLEEP 0  // ns of __nanosleep between failed mbarrier polls (0: spin)
#endif
constexpr int kWsProducers = WS_PRODUCERS;
constexpr int kWsThreads = (kWsConsumers + kWsProducers) * 32;

struct WsStage {
    WarpStage blk[kWsConsumers];
    uint32_t cnt[kWsConsumers];
    uint32_t last;  // no stage follows this one
};

#ifndef WS_RAW
#define WS_RAW 2
#endif
// producer's gather ring (batches in flight + 1).  One batch ahead is enough:
// the records were just written by K3 and are L2-resident; a deeper ring only
// costs shared memory (2 / 3 / 4: 3010 / 2963 / 2909 frames/s on the cfg-3 path)
constexpr int kWsRaw = WS_RAW;
struct WsRaw {
    double2 m[32];
    float4 q0[32], col[32];
    float2 h[32];
    uint32_t gid[32];
};

struct WsShared {
    WsStage st[kWsStages];
    WsRaw raw[kWsProducers][kWsRaw];
    unsigned long long full[kWsStages], empty[kWsStages];
    uint32_t done_warps;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(
                     smem_addr(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
#if WS_SLEEP
    uint32_t ok = 0;
    while (true) {
        asm volatile(
            "{ .reg .pred p;\n"
            "  mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "  selp.u32 %0, 1, 0, p;\n"
            "}"
            : "=r"(ok)
            : "r"(smem_addr(b)), "r"(parity)
            : "memory");
        if (ok) break;
        __nanosleep(WS_SLEEP);
    }
#elif WS_HINT
    // suspend-time hint: the warp sleeps in hardware until the phase flips
    // (or the hint expires) instead of re-issuing the poll
    asm volatile(
        "{ .reg .pred p;\n"
        "WAIT_%=:\n"
        "  mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "  @!p bra WAIT_%=;\n"
        "}" ::"r"(smem_addr(b)),
        "r"(parity), "n"(WS_HINT)
        : "memory");
#else
    asm volatile(
        "{ .reg .pred p;\n"
        "WAIT_%=:\n"
        "  mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "  @!p bra WAIT_%=;\n"
        "}" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
#endif
}

#ifndef WS_MIN_CTAS
#define WS_MIN_CTAS 3
#endif
__global__ void __launch_bounds__(kWsThreads, WS_MIN_CTAS) k_blend_ws(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ order,
    const unsigned long long* __restrict__ keys, const Gauss64* __restrict__ g64,
    const Gauss32* __restrict__ g32, const int width, const int height, const int tiles_x,
    float* __restrict__ image) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char ws_raw[];
    WsShared& sh = *reinterpret_cast<WsShared*>(ws_raw);
    const int tile = int(order[blockIdx.x]);  // heaviest tiles first
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tx0 = (tile % tiles_x) * kTile, ty0 = (tile / tiles_x) * kTile;
    const uint32_t b = offsets[tile], e = offsets[tile + 1];
    if (threadIdx.x == 0) {
        for (int s = 0; s < kWsStages; ++s) {
            mbar_init(&sh.full[s], 32);  // one producer warp fills a stage
            mbar_init(&sh.empty[s], kWsConsumers * 32);
        }
        sh.done_warps = 0;
    }
    __syncthreads();

    if (warp >= kWsConsumers) {
        // ---------------- producers ----------------
        // Producer p fills the stages of batches p, p + 2, p + 4, ...  Records
        // are gathered with cp.async into a private ring kWsRaw of its batches
        // ahead (keys one batch further, in registers).  A splat's blocks are
        // the ones its alpha box overlaps: one range test per axis, then one
        // ballot per block to compact the hits in pair order.
        const uint32_t pid = warp - kWsConsumers;
        constexpr uint32_t kNone = 0xFFFFFFFFu;
        auto batch_base = [&](uint32_t j) { return b + 32u * (pid + kWsProducers * j); };
        auto load_key = [&](uint32_t j) -> uint32_t {
            const uint32_t at = batch_base(j);
            return at + lane < e ? uint32_t(keys[at + lane]) : kNone;
        };
        auto gather = [&](uint32_t gi, int slot) {
            WsRaw& r = sh.raw[pid][slot];
            r.gid[lane] = gi;
            if (gi != kNone) {
                cp_async16(&r.m[lane], &g32[gi].mx);
                cp_async16(&r.q0[lane], &g32[gi].ha);
                cp_async16(&r.col[lane], &g32[gi].op);
                cp_async8(&r.h[lane], &g32[gi].hx);
            }
            cp_async_commit();
        };
#pragma unroll
        for (int j = 0; j < kWsRaw - 1; ++j) gather(load_key(j), j);
        uint32_t gi_ahead = load_key(kWsRaw - 1);
        const unsigned lt = (1u << lane) - 1u;
        for (uint32_t j = 0;; ++j) {
            const uint32_t i = pid + kWsProducers * j;  // global batch index
            const uint32_t base = batch_base(j);
            gather(gi_ahead, int((j + kWsRaw - 1) % kWsRaw));
            gi_ahead = load_key(j + kWsRaw);
            cp_async_wait<kWsRaw - 1>();  // batch j of this producer has landed
            __syncwarp();
            const WsRaw& r = sh.raw[pid][j % kWsRaw];
            const int s = int(i % kWsStages);
            const uint32_t use = i / kWsStages;
            if (use > 0) mbar_wait(&sh.empty[s], (use - 1) & 1u);
            WsStage& st = sh.st[s];
            const bool stop = base >= e || (!WS_NOSTOP && *(volatile uint32_t*)&sh.done_warps == kWsConsumers);
            if (!stop) {
                const uint32_t gi = r.gid[lane];
                const double2 m = r.m[lane];
                const float4 q0 = r.q0[lane], col = r.col[lane];
                const float2 h = r.h[lane];
                // tile-relative box; block (bxi, byi) spans pixel centres
                // [8 bxi + 0.5, 8 bxi + 7.5] x [4 byi + 0.5, 4 byi + 3.5]
                float mtx = 0.f, mty = 0.f;
                unsigned xm = 0, ym = 0;  // overlapped block columns / rows
                if (gi != kNone && h.x >= 0.0f) {
                    mtx = float(m.x - double(tx0));
                    mty = float(m.y - double(ty0));
                    xm = (mtx - h.x <= 7.5f && mtx + h.x >= 0.5f ? 1u : 0u) |
                         (mtx - h.x <= 15.5f && mtx + h.x >= 8.5f ? 2u : 0u);
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        ym |= (mty - h.y <= 4.0f * v + 3.5f && mty + h.y >= 4.0f * v + 0.5f)
                                  ? (1u << v)
                                  : 0u;
                }
#pragma unroll
                for (int w = 0; w < kWsConsumers; ++w) {
                    const bool hit = ((xm >> (w & 1)) & 1u) && ((ym >> (w >> 1)) & 1u);
                    const unsigned bits = __ballot_sync(0xffffffffu, hit);
                    if (hit) {
                        const int slot = __popc(bits & lt);
                        // block-relative mean, rounded from the FP64 mean exactly as k_blend_fast
#if WS_FASTMEAN  // timing experiment only: not the certified rounding
                        const float mlx = mtx - float((w & 1) * 8);
                        const float mly = mty - float((w >> 1) * 4);
#else
                        const float mlx = float(m.x - double(tx0 + (w & 1) * 8));
                        const float mly = float(m.y - double(ty0 + (w >> 1) * 4));
#endif
                        st.blk[w].geo[slot] = make_float4(mlx, mly, q0.x, q0.z);
                        st.blk[w].ct[slot] = make_float4(q0.y, q0.w, col.x, col.y);
                        st.blk[w].gb[slot] = make_float2(col.z, col.w);
                        st.blk[w].gid[slot] = gi;
                    }
                    if (lane == 0) st.cnt[w] = __popc(bits);
                }
            } else if (lane < kWsConsumers) {
                st.cnt[lane] = 0;
            }
            const bool last = stop || base + 32 >= e;
            if (lane == 0) st.last = last ? 1u : 0u;
            __syncwarp();
            mbar_arrive(&sh.full[s]);
            if (last) break;
        }
        cp_async_wait<0>();  // no gather may land after the CTA retires
        return;
    }

    // ---------------- consumers: warp w owns the 8x4 block (w & 1, w >> 1) ----
    const int bx = tx0 + int(warp & 1) * 8, by = ty0 + int(warp >> 1) * 4;
    const int x = bx + int(lane & 7), y = by + int(lane >> 3);
    const bool inside = x < width && y < height;
    const float pxl = float(lane & 7) + 0.5f, pyl = float(lane >> 3) + 0.5f;
    const double px = double(x) + 0.5, py = double(y) + 0.5;
    PixState pix{inside ? 1.0f : 0.0f, 0.0f, 0.0f, 0.0f};  // T == 0: nothing to do
    bool counted = false;
    for (uint32_t i = 0;; ++i) {
        const int s = int(i % kWsStages);
        mbar_wait(&sh.full[s], (i / kWsStages) & 1u);
        const WarpStage& st = sh.st[s].blk[warp];
        const int nh = int(sh.st[s].cnt[warp]);
        const bool last = sh.st[s].last != 0;
        if (!WS_NOCONSUME && nh > 0 && __any_sync(0xffffffffu, pix.T != 0.0f)) {
            const PixState saved = pix;
            bool unsure = false;
            int k = 0;
            for (; k + 2 <= nh; k += 2) {
                blend_sample_fast(st, k, pxl, pyl, pix, unsure);
                blend_sample_fast(st, k + 1, pxl, pyl, pix, unsure);
            }
            if (k < nh) blend_sample_fast(st, k, pxl, pyl, pix, unsure);
            if (__any_sync(0xffffffffu, unsure)) {  // rare: certified FP64 decisions
                pix = saved;
                for (int j = 0; j < nh; ++j)
                    blend_sample_checked(st, j, pxl, pyl, px, py, g64, g32, pix);
            }
        }
        __syncwarp();
        mbar_arrive(&sh.empty[s]);
        if (!counted && __all_sync(0xffffffffu, pix.T == 0.0f)) {
            counted = true;
            if (lane == 0) atomicAdd(&sh.done_warps, 1u);
        }
        if (last) break;
    }
    if (inside) {
        float* o = image + (size_t(y) * width + x) * 3;
        o[0] = pix.cr;
        o[1] = pix.cg;
        o[2] = pix.cb;
    }
}

// ---------------------------------------------------------------------------
// Persistent form of k_blend_ws: one CTA per resident slot walks the tiles
// blockIdx.x, blockIdx.x + G, ... of the heavy-first order.  The stage ring
// runs across tile boundaries, so the producers gather the next tile's first
// batches while the consumers still blend the current one (no per-tile CTA
// start-up, no drained pipeline at tile ends).  A tile contributes
// max(1, ceil(n / 32)) stages; producer p fills the CTA's global stages p, p + 2,
// ...; a stage carries its tile and flags (last stage of the tile: consumers
// store their pixels and start over; last stage of the CTA).
struct WspStage {
    WarpStage blk[kWsConsumers];
    uint32_t cnt[kWsConsumers];
    int x0, y0;      // pixel origin of the stage's tile
    uint32_t flags;  // 1: last stage of its tile, 2: last stage of the CTA
};
constexpr int kTq = 16;  // tile-queue ring (producer 0's cursor runs <= 12 tiles ahead)
struct WspShared {
    WspStage st[kWsStages];
    WsRaw raw[kWsProducers][kWsRaw];
    unsigned long long full[kWsStages], empty[kWsStages];
    unsigned long long tq[kTq];  // (k << 32) | tile, see wsp_tile
};

// Position in a CTA's stage sequence: k-th tile of the CTA, batch bi of it.
// The next tile's bucket bounds and the tile after it are loaded one tile
// ahead, so crossing a tile boundary never waits on a dependent global load
// (order -> offsets -> keys would be three round trips in the producer loop).
#ifndef WSP_SNAKE
#define WSP_SNAKE 1
#endif
#ifndef WSP_DYNAMIC
#define WSP_DYNAMIC 1  // tiles from the frame's ticket queue (else static slots)
#endif
struct TileCur {
    uint32_t k, bi, b, e, nb;
    int tile;  // -1: past the CTA's last tile
    int tx0, ty0;
    int ntile, nntile;  // tiles k + 1, k + 2 (-1: none)
    uint32_t nb_b, nb_e;  // bucket of tile k + 1
};
// boustrophedon over the heavy-first order: CTA c takes the c-th tile of even
// rounds and the (G-1-c)-th of odd ones, so no CTA always draws the heaviest
// tile of each round
__device__ __forceinline__ uint32_t wsp_slot(uint32_t k) {
    return k * gridDim.x +
           ((WSP_SNAKE && (k & 1u)) ? gridDim.x - 1u - blockIdx.x : blockIdx.x);
}
// The CTA's k-th tile.  Dynamic (ticket != null): tiles are taken from the
// frame's queue in heavy-first order; producer 0's look-ahead cursor takes the
// ticket and publishes the tile in a shared ring, every other cursor reads it
// there (waiting for producer 0 if it is ahead -- producer 0 never waits on
// producer 1, so this cannot deadlock).  Static: the boustrophedon slot.
struct WspSrc {
    const uint32_t* order;
    uint32_t n_tiles;
    unsigned* ticket;
    WspShared* sh;
};
__device__ __forceinline__ int wsp_tile(uint32_t k, const WspSrc& src, bool fetch) {
    if (!src.ticket) {
        const uint32_t slot = wsp_slot(k);
        return slot < src.n_tiles ? int(src.order[slot]) : -1;
    }
    // one 64-bit word per ring entry, (k << 32) | tile, written and read with
    // shared-memory atomics: the reader either sees entry k whole or keeps waiting
    const uint32_t q = k % kTq;
    unsigned long long* ent = &src.sh->tq[q];
    if (fetch) {
        uint32_t t = 0;
        if ((threadIdx.x & 31) == 0) t = atomicAdd(src.ticket, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        const int tile = t < src.n_tiles ? int(src.order[t]) : -1;
        if ((threadIdx.x & 31) == 0) atomicExch(ent, (unsigned long long)k << 32 | uint32_t(tile));
        __syncwarp();
        return tile;
    }
    unsigned long long v = 0;
    if ((threadIdx.x & 31) == 0)
        do {
            v = atomicOr(ent, 0ull);
        } while (uint32_t(v >> 32) != k);
    return int(uint32_t(__shfl_sync(0xffffffffu, (unsigned long long)v, 0)));
}
__device__ __forceinline__ void tile_cur_enter(TileCur& c, int tiles_x) {
    c.bi = 0;
    if (c.tile < 0) {
        c.b = c.e = 0;
        c.nb = 1;
        return;
    }
    c.tx0 = (c.tile % tiles_x) * kTile;
    c.ty0 = (c.tile / tiles_x) * kTile;
    c.nb = c.e > c.b ? (c.e - c.b + 31u) / 32u : 1u;
}
__device__ __forceinline__ void tile_cur_init(TileCur& c, const WspSrc& src, bool fetch,
                                              const uint32_t* offsets, int tiles_x) {
    c.k = 0;
    c.tile = wsp_tile(0, src, fetch);
    c.ntile = wsp_tile(1, src, fetch);
    c.nntile = wsp_tile(2, src, fetch);
    if (c.tile >= 0) {
        c.b = offsets[c.tile];
        c.e = offsets[c.tile + 1];
    }
    if (c.ntile >= 0) {
        c.nb_b = offsets[c.ntile];
        c.nb_e = offsets[c.ntile + 1];
    }
    tile_cur_enter(c, tiles_x);
}
__device__ __forceinline__ void tile_cur_step(TileCur& c, uint32_t n, const WspSrc& src,
                                              bool fetch, const uint32_t* offsets, int tiles_x) {
    c.bi += n;
    while (c.tile >= 0 && c.bi >= c.nb) {
        const uint32_t over = c.bi - c.nb;
        ++c.k;
        c.tile = c.ntile;
        c.b = c.nb_b;
        c.e = c.nb_e;
        c.ntile = c.nntile;
        if (c.ntile >= 0) {  // loaded a tile ago
            c.nb_b = offsets[c.ntile];
            c.nb_e = offsets[c.ntile + 1];
        }
        c.nntile = wsp_tile(c.k + 2, src, fetch);
        tile_cur_enter(c, tiles_x);
        c.bi = over;
    }
}

__global__ void __launch_bounds__(kWsThreads, WS_MIN_CTAS) k_blend_wsp(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ order,
    const unsigned long long* __restrict__ keys, const Gauss64* __restrict__ g64,
    const Gauss32* __restrict__ g32, const int width, const int height, const int tiles_x,
    const uint32_t n_tiles, unsigned* ticket, float* __restrict__ image) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char ws_raw[];
    WspShared& sh = *reinterpret_cast<WspShared*>(ws_raw);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kWsStages; ++s) {
            mbar_init(&sh.full[s], 32);
            mbar_init(&sh.empty[s], kWsConsumers * 32);
        }
    }
    if (threadIdx.x < kTq) sh.tq[threadIdx.x] = ~0ull;
    __syncthreads();

    if (warp >= kWsConsumers) {
        // ---------------- producers ----------------
        const uint32_t pid = warp - kWsConsumers;
        constexpr uint32_t kNone = 0xFFFFFFFFu;
        auto load_key = [&](const TileCur& c) -> uint32_t {
            const uint32_t at = c.b + 32u * c.bi + lane;
            return (c.tile >= 0 && at < c.e) ? uint32_t(keys[at]) : kNone;
        };
        auto gather = [&](uint32_t gi, int slot) {
            WsRaw& r = sh.raw[pid][slot];
            r.gid[lane] = gi;
            if (gi != kNone) {
                cp_async16(&r.m[lane], &g32[gi].mx);
                cp_async16(&r.q0[lane], &g32[gi].ha);
                cp_async16(&r.col[lane], &g32[gi].op);
                cp_async8(&r.h[lane], &g32[gi].hx);
            }
            cp_async_commit();
        };
        const WspSrc src{order, n_tiles, ticket, &sh};
        const bool lead = pid == 0;  // producer 0's look-ahead cursor takes the tickets
        TileCur cg;  // the stage whose key is loaded next
        tile_cur_init(cg, src, lead, offsets, tiles_x);
        tile_cur_step(cg, pid, src, lead, offsets, tiles_x);
        TileCur cp;  // the stage being filled
        tile_cur_init(cp, src, false, offsets, tiles_x);
        tile_cur_step(cp, pid, src, false, offsets, tiles_x);
        if (pid == 0 && cp.tile < 0) {
            // the queue was empty when this CTA started: one empty final stage
            // releases the consumers
            WspStage& st = sh.st[0];
            if (lane < kWsConsumers) st.cnt[lane] = 0;
            if (lane == 0) {
                st.x0 = st.y0 = 0;
                st.flags = 2u;
            }
            __syncwarp();
            mbar_arrive(&sh.full[0]);
        }
#pragma unroll
        for (int j = 0; j < kWsRaw - 1; ++j) {
            gather(load_key(cg), j);
            tile_cur_step(cg, kWsProducers, src, lead, offsets, tiles_x);
        }
        uint32_t gi_ahead = load_key(cg);
        tile_cur_step(cg, kWsProducers, src, lead, offsets, tiles_x);
        const unsigned lt = (1u << lane) - 1u;
        for (uint32_t j = 0; cp.tile >= 0; ++j) {
            const uint32_t i = pid + kWsProducers * j;  // the CTA's global stage index
            gather(gi_ahead, int((j + kWsRaw - 1) % kWsRaw));
            gi_ahead = load_key(cg);
            tile_cur_step(cg, kWsProducers, src, lead, offsets, tiles_x);
            cp_async_wait<kWsRaw - 1>();
            __syncwarp();
            const WsRaw& r = sh.raw[pid][j % kWsRaw];
            const int s = int(i % kWsStages);
            const uint32_t use = i / kWsStages;
            if (use > 0) mbar_wait(&sh.empty[s], (use - 1) & 1u);
            WspStage& st = sh.st[s];
            const int tx0 = cp.tx0, ty0 = cp.ty0;
            const uint32_t gi = r.gid[lane];
            const double2 m = r.m[lane];
            const float4 q0 = r.q0[lane], col = r.col[lane];
            const float2 h = r.h[lane];
            float mtx = 0.f, mty = 0.f;
            unsigned xm = 0, ym = 0;
            if (gi != kNone && h.x >= 0.0f) {
                mtx = float(m.x - double(tx0));
                mty = float(m.y - double(ty0));
                xm = (mtx - h.x <= 7.5f && mtx + h.x >= 0.5f ? 1u : 0u) |
                     (mtx - h.x <= 15.5f && mtx + h.x >= 8.5f ? 2u : 0u);
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    ym |= (mty - h.y <= 4.0f * v + 3.5f && mty + h.y >= 4.0f * v + 0.5f)
                              ? (1u << v)
                              : 0u;
            }
#pragma unroll
            for (int w = 0; w < kWsConsumers; ++w) {
                const bool hit = ((xm >> (w & 1)) & 1u) && ((ym >> (w >> 1)) & 1u);
                const unsigned bits = __ballot_sync(0xffffffffu, hit);
                if (hit) {
                    const int slot = __popc(bits & lt);
                    const float mlx = float(m.x - double(tx0 + (w & 1) * 8));
                    const float mly = float(m.y - double(ty0 + (w >> 1) * 4));
                    st.blk[w].geo[slot] = make_float4(mlx, mly, q0.x, q0.z);
                    st.blk[w].ct[slot] = make_float4(q0.y, q0.w, col.x, col.y);
                    st.blk[w].gb[slot] = make_float2(col.z, col.w);
                    st.blk[w].gid[slot] = gi;
                }
                if (lane == 0) st.cnt[w] = __popc(bits);
            }
            const bool tile_end = cp.bi + 1 >= cp.nb;
            const bool cta_end = tile_end && cp.ntile < 0;
            if (lane == 0) {
                st.x0 = tx0;
                st.y0 = ty0;
                st.flags = (tile_end ? 1u : 0u) | (cta_end ? 2u : 0u);
            }
            __syncwarp();
            mbar_arrive(&sh.full[s]);
            tile_cur_step(cp, kWsProducers, src, false, offsets, tiles_x);
        }
        cp_async_wait<0>();  // no gather may land after the CTA retires
        return;
    }

    // ---------------- consumers: warp w owns the 8x4 block (w & 1, w >> 1) ----
    const float pxl = float(lane & 7) + 0.5f, pyl = float(lane >> 3) + 0.5f;
    PixState pix{1.0f, 0.0f, 0.0f, 0.0f};
    for (uint32_t i = 0;; ++i) {
        const int s = int(i % kWsStages);
        mbar_wait(&sh.full[s], (i / kWsStages) & 1u);
        const WarpStage& st = sh.st[s].blk[warp];
        const int nh = int(sh.st[s].cnt[warp]);
        const uint32_t flags = sh.st[s].flags;
        const int x = sh.st[s].x0 + int(warp & 1) * 8 + int(lane & 7);
        const int y = sh.st[s].y0 + int(warp >> 1) * 4 + int(lane >> 3);
        if (!WS_NOCONSUME && nh > 0 && __any_sync(0xffffffffu, pix.T != 0.0f)) {
            const PixState saved = pix;
            bool unsure = false;
            int k = 0;
            for (; k + 2 <= nh; k += 2) {
                blend_sample_fast(st, k, pxl, pyl, pix, unsure);
                blend_sample_fast(st, k + 1, pxl, pyl, pix, unsure);
            }
            if (k < nh) blend_sample_fast(st, k, pxl, pyl, pix, unsure);
            if (__any_sync(0xffffffffu, unsure)) {  // rare: certified FP64 decisions
                pix = saved;
                const double px = double(x) + 0.5, py = double(y) + 0.5;
                for (int j = 0; j < nh; ++j)
                    blend_sample_checked(st, j, pxl, pyl, px, py, g64, g32, pix);
            }
        }
        __syncwarp();
        mbar_arrive(&sh.empty[s]);
        if (flags & 1u) {
            if (x < width && y < height) {
                float* o = image + (size_t(y) * width + x) * 3;
                o[0] = pix.cr;
                o[1] = pix.cg;
                o[2] = pix.cb;
            }
            pix = PixState{1.0f, 0.0f, 0.0f, 0.0f};
        }
        if (flags & 2u) break;
    }
}

// ---------------------------------------------------------------------------
// TMA-staged blend (north_star (4)).  Two kernels:
//
// K6a k_pack_blend -- after the sort, every pair p gets a 48-byte blend record
//     written at p, i.e. each tile's records are contiguous and in blend
//     order: the splat's tile-relative mean (rounded once from FP64, as the
//     warp-block means were), its log2e-scaled conic, threshold, opacity,
//     colour, the 8-bit mask of the tile's 8x4 blocks its alpha box overlaps
//     (the cull of the old producer warps, done once per pair in a flat,
//     fully parallel pass) and its slot (for the rare FP64 re-check).
// K6b k_blend_tma -- persistent, one producer thread + 8 consumer warps per
//     CTA.  The producer takes tiles from the frame's ticket queue (heavy-first
//     order) and streams each tile's records into a ring of shared-memory
//     stages with one cp.async.bulk per 32-record chunk (mbarrier complete_tx);
//     it holds no registers for the data and runs up to kTmaStages chunks
//     ahead, across tile boundaries.  Consumer warp w owns the 8x4 block
//     (w & 1, w >> 1): it takes its hits from the mask bits of the chunk (one
//     ballot), blends them in pair order in FP32 (the certified skip test of
//     k_blend_ws; a batch with an uncertain sample is re-run with the FP64
//     decision), and frees the stage with one mbarrier arrive per warp.  When
//     all 8 warps of a tile have terminated (T < 1e-4 everywhere) the producer
//     stops streaming that tile.


__global__ void __launch_bounds__(128) k_pack_blend(const uint32_t* __restrict__ offsets,
                                                    const unsigned long long* __restrict__ keys,
                                                    const Gauss64* __restrict__ g64,
                                                    const Gauss32* __restrict__ g32,
                                                    const int tiles_x, BlendRec* __restrict__ rec) {
    pdl_wait();
    pdl_trigger();
    const int tile = blockIdx.x;
    const uint32_t b = offsets[tile], e = offsets[tile + 1];
    const int tx0 = (tile % tiles_x) * kTile, ty0 = (tile / tiles_x) * kTile;
    for (uint32_t p = b + threadIdx.x; p < e; p += blockDim.x)
        rec[p] = make_blend_rec(g64, g32, uint32_t(keys[p]), tx0, ty0);
}

#ifndef TMA_STAGES
#define TMA_STAGES 12
#endif
#ifndef TMA_COMPACT
#define TMA_COMPACT 1  // consumers compact their hits into a per-warp list (else bit scan)
#endif
#ifndef TMA_MIN_CTAS
#define TMA_MIN_CTAS 3
#endif
constexpr int kTmaStages = TMA_STAGES;
constexpr int kTmaConsumers = 8;
constexpr int kTmaThreads = (kTmaConsumers + 1) * 32;
constexpr int kDoneRing = 32;  // > kTmaStages: a tile has >= 1 stage
constexpr int kTmaChunk = 32;  // records per stage

struct TmaHdr {
    int x0, y0;
    uint32_t n;      // records in the stage (0: none)
    uint32_t flags;  // 1: last stage of its tile, 2: end of the CTA's work
};
struct TmaShared {
    BlendRec rec[kTmaStages][kTmaChunk];
#if TMA_COMPACT
    WarpStage wl[kTmaConsumers];  // per consumer warp: its hits of the current stage
#endif
    TmaHdr hdr[kTmaStages];
    unsigned long long full[kTmaStages], empty[kTmaStages];
    uint32_t done[kDoneRing];  // (tile seq << 4) | consumer warps terminated
};

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(
                     smem_addr(b)),
                 "r"(bytes)
                 : "memory");
}
// one bulk copy global -> this CTA's shared memory, completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

#ifndef TMA_PROD_HINT
#define TMA_PROD_HINT 20000  // ns: the producer sleeps in hardware on a busy ring
#endif
#ifndef TMA_CONS_HINT
#define TMA_CONS_HINT 0  // ns suspend hint of the consumers' full-barrier waits (0: spin)
#endif
// mbarrier wait with a suspend-time hint: the thread is descheduled until the
// phase completes (or the hint expires) instead of re-issuing the poll
// one poll of the phase (no blocking)
__device__ __forceinline__ bool mbar_try(unsigned long long* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p;\n"
        "  mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "  selp.u32 %0, 1, 0, p;\n"
        "}"
        : "=r"(ok)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

template <int kHintNs>
__device__ __forceinline__ void mbar_wait_hint(unsigned long long* b, uint32_t parity) {
    if (kHintNs == 0) {
        mbar_wait(b, parity);
        return;
    }
    asm volatile(
        "{ .reg .pred p;\n"
        "WAITH_%=:\n"
        "  mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "  @!p bra WAITH_%=;\n"
        "}" ::"r"(smem_addr(b)),
        "r"(parity), "n"(kHintNs)
        : "memory");
}

__global__ void __launch_bounds__(kTmaThreads, TMA_MIN_CTAS) k_blend_tma(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ order,
    const BlendRec* __restrict__ rec, const Gauss64* __restrict__ g64,
    const Gauss32* __restrict__ g32, const int width, const int height, const int tiles_x,
    const uint32_t n_tiles, unsigned* ticket, float* __restrict__ image) {
    pdl_wait();  // the record pack (and everything before it) is complete and visible
    pdl_trigger();
    extern __shared__ __align__(128) unsigned char tma_raw[];
    TmaShared& sh = *reinterpret_cast<TmaShared*>(tma_raw);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTmaStages; ++s) {
            mbar_init(&sh.full[s], 1);               // the producer's arrive(.expect_tx)
            mbar_init(&sh.empty[s], kTmaConsumers);  // one arrive per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kTmaConsumers) {
        // ---------------- producer: one thread ----------------
        if (lane != 0) return;
        // Tiles come through a three-deep pipeline -- ticket (atomic) -> tile id
        // (order[]) -> bucket bounds (offsets[]) -- advanced one step per tile
        // transition, so a transition never waits on a dependent global load
        // (a one-chunk tile streams in the time of one bulk copy).
        auto tile_of = [&](uint32_t t) -> int { return t < n_tiles ? int(__ldg(order + t)) : -1; };
        int tile = tile_of(atomicAdd(ticket, 1u));
        uint32_t b = tile >= 0 ? offsets[tile] : 0u, e = tile >= 0 ? offsets[tile + 1] : 0u;
        int nxt = tile_of(atomicAdd(ticket, 1u));
        uint32_t nb = nxt >= 0 ? offsets[nxt] : 0u, ne = nxt >= 0 ? offsets[nxt + 1] : 0u;
        int t2 = tile_of(atomicAdd(ticket, 1u));
        uint32_t raw3 = atomicAdd(ticket, 1u);
        uint32_t i = 0;  // stage sequence
        uint32_t k = 0;  // tile sequence of this CTA
        volatile uint32_t* done = sh.done;
        while (tile >= 0) {
            const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
            done[k % kDoneRing] = k << 4;  // published by the first stage's arrive
            for (uint32_t c = b;; c += kTmaChunk) {
                const int s = int(i % kTmaStages);
                if (i >= uint32_t(kTmaStages))
                    mbar_wait_hint<TMA_PROD_HINT>(&sh.empty[s], ((i / kTmaStages) - 1) & 1u);
                const uint32_t n = c < e ? min(uint32_t(kTmaChunk), e - c) : 0u;
                const bool last = c + kTmaChunk >= e || done[k % kDoneRing] == ((k << 4) | 8u);
                sh.hdr[s] = TmaHdr{x0, y0, n, last ? 1u : 0u};
                if (n) {
                    mbar_expect_tx(&sh.full[s], n * uint32_t(sizeof(BlendRec)));
                    bulk_g2s(&sh.rec[s][0], rec + c, n * uint32_t(sizeof(BlendRec)), &sh.full[s]);
                } else {
                    mbar_arrive(&sh.full[s]);
                }
                ++i;
                if (last) break;
            }
            ++k;
            tile = nxt;
            b = nb;
            e = ne;
            nxt = t2;
            nb = nxt >= 0 ? offsets[nxt] : 0u;
            ne = nxt >= 0 ? offsets[nxt + 1] : 0u;
            t2 = tile_of(raw3);
            raw3 = atomicAdd(ticket, 1u);
        }
        const int s = int(i % kTmaStages);
        if (i >= uint32_t(kTmaStages))
            mbar_wait_hint<TMA_PROD_HINT>(&sh.empty[s], ((i / kTmaStages) - 1) & 1u);
        sh.hdr[s] = TmaHdr{0, 0, 0u, 2u};
        mbar_arrive(&sh.full[s]);
        return;
    }

    // ---------------- consumers: warp w owns the 8x4 block (w & 1, w >> 1) ----
#if TMA_COMPACT
    WarpStage* wl = sh.wl;
#endif
    const int lx = int(warp & 1) * 8 + int(lane & 7), ly = int(warp >> 1) * 4 + int(lane >> 3);
    const float pxl = float(lx) + 0.5f, pyl = float(ly) + 0.5f;  // tile-relative pixel centre
    const uint32_t wbit = 1u << warp;
    PixState pix{0.0f, 0.0f, 0.0f, 0.0f};
    bool fresh = true, counted = false;
    int x = 0, y = 0;
    uint32_t k = 0;
    for (uint32_t i = 0;; ++i) {
        const int s = int(i % kTmaStages);
        mbar_wait_hint<TMA_CONS_HINT>(&sh.full[s], (i / kTmaStages) & 1u);
        const TmaHdr hd = sh.hdr[s];
        if (hd.flags & 2u) break;
        if (fresh) {
            x = hd.x0 + lx;
            y = hd.y0 + ly;
            pix = PixState{(x < width && y < height) ? 1.0f : 0.0f, 0.0f, 0.0f, 0.0f};
            fresh = false;
            counted = false;
        }
        const BlendRec* R = sh.rec[s];
        const bool mine = lane < hd.n && (__float_as_uint(R[lane].gbm.z) & wbit);
        const unsigned bits = __ballot_sync(0xffffffffu, mine);
        if (bits && __any_sync(0xffffffffu, pix.T != 0.0f)) {
            const PixState saved = pix;
            bool unsure = false;
#if TMA_COMPACT
            // this warp's hits, compacted in pair order into its own list
            WarpStage& st = wl[warp];
            if (mine) {
                const int at = __popc(bits & ((1u << lane) - 1u));
                st.geo[at] = R[lane].geo;
                st.ct[at] = R[lane].ct;
                st.gb[at] = make_float2(R[lane].gbm.x, R[lane].gbm.y);
                st.gid[at] = __float_as_uint(R[lane].gbm.w);
            }
            __syncwarp();
            const int nh = __popc(bits);
            int kk = 0;
            for (; kk + 2 <= nh; kk += 2) {
                blend_sample_fast(st, kk, pxl, pyl, pix, unsure);
                blend_sample_fast(st, kk + 1, pxl, pyl, pix, unsure);
            }
            if (kk < nh) blend_sample_fast(st, kk, pxl, pyl, pix, unsure);
            if (__any_sync(0xffffffffu, unsure)) {  // rare: certified FP64 decisions
                pix = saved;
                const double px = double(x) + 0.5, py = double(y) + 0.5;
                for (int j = 0; j < nh; ++j) blend_sample_checked(st, j, pxl, pyl, px, py, g64, g32, pix);
            }
#else
            unsigned bb = bits;
            while (bb) {
                const int j0 = __ffs(bb) - 1;
                bb &= bb - 1;
                sample_fast(R[j0].geo, R[j0].ct, make_float2(R[j0].gbm.x, R[j0].gbm.y), pxl, pyl,
                            pix, unsure);
                if (bb) {
                    const int j1 = __ffs(bb) - 1;
                    bb &= bb - 1;
                    sample_fast(R[j1].geo, R[j1].ct, make_float2(R[j1].gbm.x, R[j1].gbm.y), pxl,
                                pyl, pix, unsure);
                }
            }
            if (__any_sync(0xffffffffu, unsure)) {  // rare: certified FP64 decisions
                pix = saved;
                const double px = double(x) + 0.5, py = double(y) + 0.5;
                bb = bits;
                while (bb) {
                    const int j = __ffs(bb) - 1;
                    bb &= bb - 1;
                    sample_checked(R[j].geo, R[j].ct, make_float2(R[j].gbm.x, R[j].gbm.y),
                                   __float_as_uint(R[j].gbm.w), pxl, pyl, px, py, g64, g32, pix);
                }
            }
#endif
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.empty[s]);
        if (!counted && __all_sync(0xffffffffu, pix.T == 0.0f)) {
            counted = true;
            if (lane == 0) atomicAdd(&sh.done[k % kDoneRing], 1u);
        }
        if (hd.flags & 1u) {
            if (x < width && y < height) {
                float* o = image + (size_t(y) * width + x) * 3;
                o[0] = pix.cr;
                o[1] = pix.cg;
                o[2] = pix.cb;
            }
            fresh = true;
            ++k;
        }
    }
}

// ---------------------------------------------------------------------------
// TMA gather4 blend (k_blend_g4, north_star (4); measured, not the default: DESIGN.md
// 3.7).  No pack pass: the sorted keys name each pair's slot, and a tile's splat
// records are gathered straight from the slot-indexed K3 records into shared memory
// by the tensor memory accelerator -- cp.async.bulk.tensor.2d ... tile::gather4, four
// rows per instruction, one 64-byte Gauss32 row per pair (conic, threshold, opacity,
// colour, alpha box and the FP64 mean; two rows per pair with the mean read from
// Gauss64 ran at the TMA's row rate, 245 vs 211 us), completion counted on the stage's
// mbarrier.
//
// Per CTA: one producer warp + 8 consumer warps, persistent, tiles from the
// frame's ticket queue (heavy-first order).  The producer walks a chunk
// sequence (32 pairs per chunk, >= 1 chunk per tile, across tiles) with a
// register FIFO: chunk j's 32 keys are loaded kG4Ahead chunks before its
// gathers are issued, and a tile's ticket -> order -> offsets chain is spread
// over three tile transitions, so the producer never waits on a dependent
// global load.  Lane 0 arms the stage's `full` barrier with the expected
// bytes, lanes 0-7 issue one gather4 each.  Consumer warp w (8x4 block
// (w & 1, w >> 1)) culls the 32 records against its block (the alpha box,
// the FP64 mean rounded to block-relative FP32 exactly as k_blend_ws), compacts
// its hits into its own list and blends them (k_blend_ws's per-sample code);
// one mbarrier arrive per warp frees the stage.  Tuning: 20 stages, 4 CTAs per SM,
// two chunks of key look-ahead (10 / 16 / 20 stages, 3 / 4 CTAs: 211 / 202 / 198 us).
#ifndef G4_STAGES
#define G4_STAGES 20
#endif
#ifndef G4_AHEAD
#define G4_AHEAD 2
#endif
#ifndef G4_MIN_CTAS
#define G4_MIN_CTAS 4
#endif
constexpr int kG4Stages = G4_STAGES;
constexpr int kG4Ahead = G4_AHEAD;  // chunks whose keys are in flight
constexpr int kG4Threads = (kTmaConsumers + 1) * 32;


__device__ __forceinline__ void gather4(void* dst, const void* tmap, int r0, int r1, int r2,
                                        int r3, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_addr(dst)),
        "l"(tmap), "r"(smem_addr(bar)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

// One chunk of the producer's sequence (warp-uniform except `slot`).
struct G4Chunk {
    int tile;  // -1: end of the CTA's work
    uint32_t n, k;
    bool last;
    uint32_t slot;  // this lane's pair (lane < n)
};


// With G4_SWIZZLE the tensor map's 64-byte swizzle stores row R's 16-byte chunk c at
// chunk c ^ ((R >> 1) & 3): the consumers' per-lane row reads (64-byte stride) then
// spread over all banks instead of two bank groups (16-way conflicts).  The swizzle
// phase comes from smem address bits [8:7], so the rows sit in 512-byte-aligned stages.
#ifndef G4_SWIZZLE
#define G4_SWIZZLE 1
#endif
struct __align__(512) G4Stage {
    float rec[8][64];  // gather4 group q: rows 4q..4q+3 (16 floats each)
};
struct G4Shared {
    G4Stage st[kG4Stages];
    uint32_t slot[kG4Stages][32];
    WarpStage wl[kTmaConsumers];
    TmaHdr hdr[kG4Stages];
    unsigned long long full[kG4Stages], empty[kG4Stages];
    uint32_t done[kDoneRing];
};
constexpr uint32_t kG4GroupBytes = 4 * 64;

__global__ void __launch_bounds__(kG4Threads, G4_MIN_CTAS) k_blend_g4(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ order,
    const unsigned long long* __restrict__ keys, const __grid_constant__ CUtensorMap map32,
    const Gauss64* __restrict__ g64, const Gauss32* __restrict__ g32, const int width,
    const int height, const int tiles_x, const uint32_t n_tiles, unsigned* ticket,
    float* __restrict__ image) {
    pdl_wait();  // the sort (and everything before it) is complete and visible
    pdl_trigger();
    extern __shared__ __align__(1024) unsigned char g4_raw[];
    G4Shared& sh = *reinterpret_cast<G4Shared*>(g4_raw);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kG4Stages; ++s) {
            mbar_init(&sh.full[s], 1);
            mbar_init(&sh.empty[s], kTmaConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kTmaConsumers) {
        // ---------------- producer warp ----------------
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map32) : "memory");
        // tile pipeline: raw ticket (lane 0) -> tile id -> bounds -> current
        auto take = [&]() -> uint32_t { return lane == 0 ? atomicAdd(ticket, 1u) : 0u; };
        auto tile_of = [&](uint32_t raw) -> int {
            const uint32_t t = __shfl_sync(0xffffffffu, raw, 0);
            return t < n_tiles ? int(__ldg(order + t)) : -1;
        };
        int cur = tile_of(take());
        uint32_t cb = cur >= 0 ? offsets[cur] : 0u, ce = cur >= 0 ? offsets[cur + 1] : 0u;
        int nxt = tile_of(take());
        uint32_t nb = nxt >= 0 ? offsets[nxt] : 0u, ne = nxt >= 0 ? offsets[nxt + 1] : 0u;
        int t2 = tile_of(take());  // bounds loaded at the next transition
        uint32_t raw3 = take();    // tile id looked up at the next transition
        uint32_t gc = cb, gk = 0;  // generator cursor: next chunk start, tile sequence
        auto gen = [&]() -> G4Chunk {
            G4Chunk ch;
            ch.tile = cur;
            ch.k = gk;
            if (cur < 0) {
                ch.n = 0;
                ch.last = true;
                ch.slot = 0;
                return ch;
            }
            ch.n = gc < ce ? min(32u, ce - gc) : 0u;
            ch.last = gc + 32u >= ce;
            ch.slot = lane < ch.n ? uint32_t(keys[gc + lane]) : 0xFFFFFFFFu;
            if (ch.last) {  // tile transition: shift the tile pipeline by one
                cur = nxt;
                cb = nb;
                ce = ne;
                nxt = t2;
                nb = nxt >= 0 ? offsets[nxt] : 0u;
                ne = nxt >= 0 ? offsets[nxt + 1] : 0u;
                t2 = tile_of(raw3);
                raw3 = take();
                gc = cb;
                ++gk;
            } else {
                gc += 32u;
            }
            return ch;
        };
        G4Chunk fifo[kG4Ahead];
#pragma unroll
        for (int j = 0; j < kG4Ahead; ++j) fifo[j] = gen();
        uint32_t i = 0;                 // stage sequence
        uint32_t killed = 0xFFFFFFFFu;  // tile sequence whose remaining chunks are dropped
        bool first_chunk = true;        // the next issued chunk starts a tile
        volatile uint32_t* done = sh.done;
        bool finished = false;
        // the loop body unrolled over the FIFO slots: no register copy of a key whose
        // load is still in flight (k_blend_cpa)
        while (!finished) {
#pragma unroll
        for (int jf = 0; jf < kG4Ahead; ++jf) {
            if (finished) break;
            const G4Chunk ch = fifo[jf];
            fifo[jf] = gen();
            if (ch.tile >= 0 && ch.k == killed) continue;  // rest of a terminated tile
            const int s = int(i % kG4Stages);
            if (i >= uint32_t(kG4Stages))
                mbar_wait_hint<TMA_PROD_HINT>(&sh.empty[s], ((i / kG4Stages) - 1) & 1u);
            ++i;
            if (ch.tile < 0) {  // the CTA's work is done
                if (lane == 0) {
                    sh.hdr[s] = TmaHdr{0, 0, 0u, 2u};
                    mbar_arrive(&sh.full[s]);
                }
                finished = true;
                continue;
            }
            // first chunk of a tile: reset its terminated-warp counter (published
            // to the consumers by this stage's arrive)
            if (first_chunk && lane == 0) done[ch.k % kDoneRing] = ch.k << 4;
            bool last = ch.last;
            if (!first_chunk && !last && done[ch.k % kDoneRing] == ((ch.k << 4) | 8u)) {
                last = true;
                killed = ch.k;
            }
            G4Stage& st = sh.st[s];
            // lanes past n name a valid row (lane 0's): their bytes are fetched, never read
            const uint32_t s0 = __shfl_sync(0xffffffffu, ch.slot, 0);
            const uint32_t slot = lane < ch.n ? ch.slot : s0;
            sh.slot[s][lane] = slot;
            const uint32_t groups = (ch.n + 3u) >> 2;
            const int q = int(lane & 7);
            const int r0 = int(__shfl_sync(0xffffffffu, slot, 4 * q + 0));
            const int r1 = int(__shfl_sync(0xffffffffu, slot, 4 * q + 1));
            const int r2 = int(__shfl_sync(0xffffffffu, slot, 4 * q + 2));
            const int r3 = int(__shfl_sync(0xffffffffu, slot, 4 * q + 3));
            if (lane == 0) {
                const int tx0 = (ch.tile % tiles_x) * kTile, ty0 = (ch.tile / tiles_x) * kTile;
                sh.hdr[s] = TmaHdr{tx0, ty0, ch.n, last ? 1u : 0u};
            }
            __syncwarp();
            if (lane == 0) {
                if (groups) mbar_expect_tx(&sh.full[s], groups * kG4GroupBytes);
                else mbar_arrive(&sh.full[s]);
            }
            __syncwarp();
            if (uint32_t(q) < groups && lane < 8)
                gather4(&st.rec[q][0], &map32, r0, r1, r2, r3, &sh.full[s]);
            first_chunk = last;
        }
        }
        return;
    }

    // ---------------- consumers: warp w owns the 8x4 block (w & 1, w >> 1) ----
    WarpStage& wl = sh.wl[warp];
    const float pxl = float(lane & 7) + 0.5f, pyl = float(lane >> 3) + 0.5f;  // block-relative
    const int bxo = int(warp & 1) * 8, byo = int(warp >> 1) * 4;
    PixState pix{0.0f, 0.0f, 0.0f, 0.0f};
    bool fresh = true, counted = false;
    int bx = 0, by = 0;
    uint32_t k = 0;
    const unsigned lt = (1u << lane) - 1u;
    for (uint32_t i = 0;; ++i) {
        const int s = int(i % kG4Stages);
        mbar_wait_hint<TMA_CONS_HINT>(&sh.full[s], (i / kG4Stages) & 1u);
        const TmaHdr hd = sh.hdr[s];
        if (hd.flags & 2u) break;
        if (fresh) {
            bx = hd.x0 + bxo;
            by = hd.y0 + byo;
            const int x = bx + int(lane & 7), y = by + int(lane >> 3);
            pix = PixState{(x < width && y < height) ? 1.0f : 0.0f, 0.0f, 0.0f, 0.0f};
            fresh = false;
            counted = false;
        }
        const G4Stage& st = sh.st[s];
        // this lane's row (row lane of the stage) and its chunks' physical positions
        const float* row = &st.rec[0][0] + lane * 16;
        const unsigned sw = G4_SWIZZLE ? (lane >> 1) & 3u : 0u;
        auto chunk = [&](unsigned c) { return row + 4 * (c ^ sw); };
        bool hit = false;
        float mlx = 0.f, mly = 0.f;
        if (lane < hd.n) {
            const float2 h = *reinterpret_cast<const float2*>(chunk(2));
            const double2 m = *reinterpret_cast<const double2*>(chunk(3));
            if (h.x >= 0.0f) {
                mlx = float(m.x - double(bx));
                mly = float(m.y - double(by));
                hit = mlx - h.x <= 7.5f && mlx + h.x >= 0.5f && mly - h.y <= 3.5f &&
                      mly + h.y >= 0.5f;
            }
        }
        const unsigned bits = __ballot_sync(0xffffffffu, hit);
        if (bits && __any_sync(0xffffffffu, pix.T != 0.0f)) {
            if (hit) {
                const int at = __popc(bits & lt);
                const float4 q0 = *reinterpret_cast<const float4*>(chunk(0));
                const float4 col = *reinterpret_cast<const float4*>(chunk(1));
                wl.geo[at] = make_float4(mlx, mly, q0.x, q0.z);
                wl.ct[at] = make_float4(q0.y, q0.w, col.x, col.y);
                wl.gb[at] = make_float2(col.z, col.w);
                wl.gid[at] = sh.slot[s][lane];
            }
            __syncwarp();
            const PixState saved = pix;
            bool unsure = false;
            const int nh = __popc(bits);
            int kk = 0;
            for (; kk + 2 <= nh; kk += 2) {
                blend_sample_fast(wl, kk, pxl, pyl, pix, unsure);
                blend_sample_fast(wl, kk + 1, pxl, pyl, pix, unsure);
            }
            if (kk < nh) blend_sample_fast(wl, kk, pxl, pyl, pix, unsure);
            if (__any_sync(0xffffffffu, unsure)) {  // rare: certified FP64 decisions
                pix = saved;
                const double px = double(bx + int(lane & 7)) + 0.5;
                const double py = double(by + int(lane >> 3)) + 0.5;
                for (int j = 0; j < nh; ++j) blend_sample_checked(wl, j, pxl, pyl, px, py, g64, g32, pix);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.empty[s]);
        if (!counted && __all_sync(0xffffffffu, pix.T == 0.0f)) {
            counted = true;
            if (lane == 0) atomicAdd(&sh.done[k % kDoneRing], 1u);
        }
        if (hd.flags & 1u) {
            const int x = bx + int(lane & 7), y = by + int(lane >> 3);
            if (x < width && y < height) {
                float* o = image + (size_t(y) * width + x) * 3;
                o[0] = pix.cr;
                o[1] = pix.cg;
                o[2] = pix.cb;
            }
            fresh = true;
            ++k;
        }
    }
}

// ---------------------------------------------------------------------------
// cp.async-staged blend (K6, the default fast kernel).  k_blend_g4's structure -- one producer warp,
// eight consumer warps that cull and compact their own hits -- with the
// records gathered by per-lane cp.async instead of TMA gather4 (whose row
// rate bounds k_blend_g4).  The producer only moves bytes: per 32-pair chunk
// it issues four cp.async per lane (the splat's FP64 mean, the FP32 conic +
// threshold, opacity + colour, alpha box: 56 B) straight into the stage and
// lets the copies themselves complete the stage's `full` barrier
// (cp.async.mbarrier.arrive.noinc), so it never waits for data and can run
// kCpaStages chunks ahead -- the deep look-ahead that k_blend_wsp could not
// afford with its 11 KB per-block stages (2 KB per stage here).  Keys are
// loaded kCpaAhead chunks before their gathers are issued.  Consumers run
// k_blend_g4's cull/compact + the certified per-sample code of k_blend_ws
// (same block-relative FP32 means, so the pixels equal k_blend_wsp's).
// Tuning (cfg-3 path, 100 strided frames, four in flight; tools/variants.sh):
// stages 8 / 12 / 16 / 20 / 22 / 24: 3,410 / 3,459 / 3,442 / 3,520 / 3,493 / 3,443
// frames/s (24 no longer fits 4 CTAs per SM); key look-ahead 2 / 3 / 5: 3,469 / 3,437 /
// 3,323; 3 / 4 / 5 CTAs per SM (72 / 56 / 40 registers): 3,379 / 3,459 / 3,364;
// cp.async.cg (L2 only) vs .ca: 3,459 vs 3,421; a 500 ns suspend hint on the
// consumers' waits: 3,448.
#ifndef CPA_STAGES
#define CPA_STAGES 20
#endif
#ifndef CPA_AHEAD
#define CPA_AHEAD 2
#endif
#ifndef CPA_MIN_CTAS
#define CPA_MIN_CTAS 4
#endif
#ifndef CPA_CONS_HINT
#define CPA_CONS_HINT 0
#endif
#ifndef CPA_CONS_SLEEP
#define CPA_CONS_SLEEP 0  // ns of __nanosleep between the consumers' polls (0: try_wait)
#endif
#ifndef CPA_CG
#define CPA_CG 1
#endif
#ifndef CPA_ROTATE
#define CPA_ROTATE 0
#endif
// 1: the copies complete the stage themselves (cp.async.mbarrier.arrive.noinc);
// 0: the producer publishes stage i - kCpaLag after cp.async.wait_group (lagged).
// Both are racecheck-clean; 1 is faster (3,517 vs 3,461 frames/s, lag 3 / 6 / 10 alike).
#ifndef CPA_ASYNC_ARRIVE
#define CPA_ASYNC_ARRIVE 1
#endif
#ifndef CPA_LAG
#define CPA_LAG 6
#endif
constexpr int kCpaLag = CPA_LAG;

// Ring depth by frame size: 20 stages at 1080p, 16 above kCpaBigFrameTiles tiles.
// At 4K (32,400 tiles) the 20-stage CTAs (4 x 51 KB of shared memory per SM) cost
// 11 % of cfg 4's frame rate against 12 or 16 stages, while at 1080p 20 stages are
// 1.5 % ahead of 12 / 16 (cfg 3 3,525 / 3,471 / 3,470, cfg 4 511 / 573 / 572 frames/s;
// chosen per frame: cfg 3 3,520-3,529, cfg 4 567-572 with 16, 562-567 with 12).
#ifndef CPA_STAGES_BIG
#define CPA_STAGES_BIG 16
#endif
constexpr int kCpaStages = CPA_STAGES;
constexpr int kCpaStagesBig = CPA_STAGES_BIG;
constexpr int kCpaBigFrameTiles = 12288;
constexpr int kCpaAhead = CPA_AHEAD;
constexpr int kCpaThreads = (kTmaConsumers + 1) * 32;
static_assert(kCpaStages < kDoneRing && kCpaStagesBig < kDoneRing, "a tile has >= 1 stage");
static_assert(kCpaLag < kCpaStages && kCpaLag < kCpaStagesBig,
              "a stage is published before the producer waits for its reuse");

struct CpaStage {
    double2 m[32];   // Gauss32 (mx, my), the FP64 mean
    float4 q0[32];   // Gauss32 (ha, cb, hc, ethr)
    float4 col[32];  // Gauss32 (op, r, g, b)
    float2 h[32];    // Gauss32 (hx, hy)
    uint32_t slot[32];
};
template <int S>
struct CpaShared {
    CpaStage st[S];
    WarpStage wl[kTmaConsumers];
    TmaHdr hdr[S];
    unsigned long long full[S], empty[S];
    uint32_t done[kDoneRing];
};

// the stage barrier counts this thread's arrival once all its earlier
// cp.async copies have landed
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(b))
                 : "memory");
}

template <int S>
__global__ void __launch_bounds__(kCpaThreads, CPA_MIN_CTAS) k_blend_cpa(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ order,
    const unsigned long long* __restrict__ keys, const Gauss64* __restrict__ g64,
    const Gauss32* __restrict__ g32, const int width, const int height, const int tiles_x,
    const uint32_t n_tiles, unsigned* ticket, float* __restrict__ image) {
    pdl_wait();  // the sort (and everything before it) is complete and visible
    pdl_trigger();
    extern __shared__ __align__(128) unsigned char cpa_raw[];
    CpaShared<S>& sh = *reinterpret_cast<CpaShared<S>*>(cpa_raw);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&sh.full[s], CPA_ASYNC_ARRIVE ? 33 : 32);  // + the header's arrive
            mbar_init(&sh.empty[s], kTmaConsumers * 32);  // every consumer lane
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kTmaConsumers) {
        // ---------------- producer warp ----------------
        auto take = [&]() -> uint32_t { return lane == 0 ? atomicAdd(ticket, 1u) : 0u; };
        auto tile_of = [&](uint32_t raw) -> int {
            const uint32_t t = __shfl_sync(0xffffffffu, raw, 0);
            return t < n_tiles ? int(__ldg(order + t)) : -1;
        };
        int cur = tile_of(take());
        uint32_t cb = cur >= 0 ? offsets[cur] : 0u, ce = cur >= 0 ? offsets[cur + 1] : 0u;
        int nxt = tile_of(take());
        uint32_t nb = nxt >= 0 ? offsets[nxt] : 0u, ne = nxt >= 0 ? offsets[nxt + 1] : 0u;
        int t2 = tile_of(take());
        uint32_t raw3 = take();
        uint32_t gc = cb, gk = 0;
        auto gen = [&]() -> G4Chunk {
            G4Chunk ch;
            ch.tile = cur;
            ch.k = gk;
            if (cur < 0) {
                ch.n = 0;
                ch.last = true;
                ch.slot = 0;
                return ch;
            }
            ch.n = gc < ce ? min(32u, ce - gc) : 0u;
            ch.last = gc + 32u >= ce;
            ch.slot = lane < ch.n ? uint32_t(keys[gc + lane]) : 0xFFFFFFFFu;
            if (ch.last) {
                cur = nxt;
                cb = nb;
                ce = ne;
                nxt = t2;
                nb = nxt >= 0 ? offsets[nxt] : 0u;
                ne = nxt >= 0 ? offsets[nxt + 1] : 0u;
                t2 = tile_of(raw3);
                raw3 = take();
                gc = cb;
                ++gk;
            } else {
                gc += 32u;
            }
            return ch;
        };
        // Chunk FIFO in registers, kCpaAhead deep.  The loop body is unrolled over the
        // FIFO slots so an entry is never copied between registers: a copy of a key whose
        // load is still in flight would stall the warp on it (one chunk of look-ahead).
        G4Chunk fifo[kCpaAhead];
#pragma unroll
        for (int j = 0; j < kCpaAhead; ++j) fifo[j] = gen();
        uint32_t i = 0;
        uint32_t killed = 0xFFFFFFFFu;
        bool first_chunk = true;
        bool finished = false;
        while (!finished) {
#pragma unroll
        for (int jf = 0; jf < kCpaAhead; ++jf) {
            if (finished) break;
            const G4Chunk ch = fifo[jf];
            fifo[jf] = gen();
            if (ch.tile >= 0 && ch.k == killed) continue;  // rest of a terminated tile
            const int s = int(i % S);
            if (i >= uint32_t(S))
                mbar_wait_hint<TMA_PROD_HINT>(&sh.empty[s], ((i / S) - 1) & 1u);
            ++i;
            if (ch.tile < 0) {  // the CTA's work is done
                if (lane == 0) sh.hdr[s] = TmaHdr{0, 0, 0u, 2u};
#if CPA_ASYNC_ARRIVE
                __syncwarp();
                cp_async_mbar_arrive(&sh.full[s]);
                if (lane == 0) mbar_arrive(&sh.full[s]);
#else
                // publish the stages still in flight, then this one
                cp_async_wait<0>();
                for (uint32_t q = i - 1 > uint32_t(kCpaLag) ? i - 1 - uint32_t(kCpaLag) : 0u;
                     q < i; ++q)
                    mbar_arrive(&sh.full[q % S]);
#endif
                finished = true;
                continue;
            }
            // the tile's terminated-warp counter: lane 0 alone touches it (the consumers
            // bump it with shared atomics), the verdict is broadcast
            bool last = ch.last;
            {
                uint32_t kill = 0u;
                if (lane == 0) {
                    if (first_chunk) atomicExch(&sh.done[ch.k % kDoneRing], ch.k << 4);
                    else if (!last) kill = atomicOr(&sh.done[ch.k % kDoneRing], 0u) == ((ch.k << 4) | 8u);
                }
                if (__shfl_sync(0xffffffffu, kill, 0)) {
                    last = true;
                    killed = ch.k;
                }
            }
            CpaStage& st = sh.st[s];
            if (lane < ch.n) {
                const uint32_t gi = ch.slot;
#if CPA_CG  // L2 only: a record is read by one tile's CTA (and rarely reused in L1)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(&st.m[lane])),
                             "l"(&g32[gi].mx) : "memory");
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(&st.q0[lane])),
                             "l"(&g32[gi].ha) : "memory");
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(&st.col[lane])),
                             "l"(&g32[gi].op) : "memory");
#else
                cp_async16(&st.m[lane], &g32[gi].mx);
                cp_async16(&st.q0[lane], &g32[gi].ha);
                cp_async16(&st.col[lane], &g32[gi].op);
#endif
                cp_async8(&st.h[lane], &g32[gi].hx);
            }
            st.slot[lane] = ch.slot;
            if (lane == 0) {
                const int tx0 = (ch.tile % tiles_x) * kTile, ty0 = (ch.tile / tiles_x) * kTile;
                sh.hdr[s] = TmaHdr{tx0, ty0, ch.n, last ? 1u : 0u};
            }
#if CPA_ASYNC_ARRIVE
            __syncwarp();
            cp_async_mbar_arrive(&sh.full[s]);
            if (lane == 0) mbar_arrive(&sh.full[s]);
#else
            // publish stage i - kCpaLag: its copies (this lane's) have landed; every lane
            // arrives for its own copies and stores (release), which compute-sanitizer's
            // racecheck can follow (it does not model cp.async-triggered arrivals)
            cp_async_commit();
            if (i > uint32_t(kCpaLag)) {
                cp_async_wait<kCpaLag>();
                mbar_arrive(&sh.full[(i - 1 - uint32_t(kCpaLag)) % S]);
            }
#endif
            first_chunk = last;
        }
        }
        cp_async_wait<0>();  // no copy may land after the CTA retires
        return;
    }

    // ---------------- consumers: warp w owns the 8x4 block (w & 1, w >> 1) ----
    WarpStage& wl = sh.wl[warp];
    const float pxl = float(lane & 7) + 0.5f, pyl = float(lane >> 3) + 0.5f;  // block-relative
    const int bxo = int(warp & 1) * 8, byo = int(warp >> 1) * 4;
    PixState pix{0.0f, 0.0f, 0.0f, 0.0f};
    bool fresh = true, counted = false;
    int bx = 0, by = 0;
    uint32_t k = 0;
    const unsigned lt = (1u << lane) - 1u;
    for (uint32_t i = 0;; ++i) {
        const int s = int(i % S);
#if CPA_CONS_SLEEP
        // back off with __nanosleep between polls: a sleeping warp issues nothing
        while (!mbar_try(&sh.full[s], (i / S) & 1u)) __nanosleep(CPA_CONS_SLEEP);
#else
        mbar_wait_hint<CPA_CONS_HINT>(&sh.full[s], (i / S) & 1u);
#endif
        const TmaHdr hd = sh.hdr[s];
        if (hd.flags & 2u) break;
        if (fresh) {
#if CPA_ROTATE
            // the CTA's k-th tile: warp w takes block (w + k) & 7, so no warp always
            // draws the same block position of every tile
            const uint32_t bw = (warp + k) & 7u;
            bx = hd.x0 + int(bw & 1u) * 8;
            by = hd.y0 + int(bw >> 1) * 4;
#else
            bx = hd.x0 + bxo;
            by = hd.y0 + byo;
#endif
            const int x = bx + int(lane & 7), y = by + int(lane >> 3);
            pix = PixState{(x < width && y < height) ? 1.0f : 0.0f, 0.0f, 0.0f, 0.0f};
            fresh = false;
            counted = false;
        }
        const CpaStage& st = sh.st[s];
        bool hit = false;
        float mlx = 0.f, mly = 0.f;
        if (lane < hd.n && !counted) {
            const float2 h = st.h[lane];
            if (h.x >= 0.0f) {
                const double2 m = st.m[lane];
                mlx = float(m.x - double(bx));
                mly = float(m.y - double(by));
                hit = mlx - h.x <= 7.5f && mlx + h.x >= 0.5f && mly - h.y <= 3.5f &&
                      mly + h.y >= 0.5f;
            }
        }
        const unsigned bits = __ballot_sync(0xffffffffu, hit);
        if (bits) {
            if (hit) {
                const int at = __popc(bits & lt);
                const float4 q0 = st.q0[lane];
                const float4 col = st.col[lane];
                wl.geo[at] = make_float4(mlx, mly, q0.x, q0.z);
                wl.ct[at] = make_float4(q0.y, q0.w, col.x, col.y);
                wl.gb[at] = make_float2(col.z, col.w);
                wl.gid[at] = st.slot[lane];
            }
            __syncwarp();
            const PixState saved = pix;
            bool unsure = false;
            const int nh = __popc(bits);
            int kk = 0;
            for (; kk + 2 <= nh; kk += 2) {
                blend_sample_fast(wl, kk, pxl, pyl, pix, unsure);
                blend_sample_fast(wl, kk + 1, pxl, pyl, pix, unsure);
            }
            if (kk < nh) blend_sample_fast(wl, kk, pxl, pyl, pix, unsure);
            if (__any_sync(0xffffffffu, unsure)) {  // rare: certified FP64 decisions
                pix = saved;
                const double px = double(bx + int(lane & 7)) + 0.5;
                const double py = double(by + int(lane >> 3)) + 0.5;
                for (int j = 0; j < nh; ++j) blend_sample_checked(wl, j, pxl, pyl, px, py, g64, g32, pix);
            }
        }
        // every lane releases its own reads of the stage (one warp instruction)
        mbar_arrive(&sh.empty[s]);
        if (!counted && __all_sync(0xffffffffu, pix.T == 0.0f)) {
            counted = true;
            if (lane == 0) atomicAdd(&sh.done[k % kDoneRing], 1u);
        }
        if (hd.flags & 1u) {
            const int x = bx + int(lane & 7), y = by + int(lane >> 3);
            if (x < width && y < height) {
                float* o = image + (size_t(y) * width + x) * 3;
                o[0] = pix.cr;
                o[1] = pix.cg;
                o[2] = pix.cb;
            }
            fresh = true;
            ++k;
        }
    }
}


// Tensor map of the 64-byte Gauss32 rows for k_blend_g4: boxes of one row.
static bool encode_row_map(const Gauss32* g32, uint64_t rows, CUtensorMap* m) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    if (!encode || rows == 0 || rows > 0xFFFFFFFFull) return false;
    const cuuint64_t d[2] = {16, rows}, st[1] = {sizeof(Gauss32)};
    const cuuint32_t b[2] = {16, 1}, e1[2] = {1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<Gauss32*>(g32), d, st, b, e1,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  G4_SWIZZLE ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kBlendThreads = 256;  // exact kernel: one CTA per 16x16 tile
constexpr int kWarps = kBlendThreads / 32;

struct BlendSmemExact {
    double4 geo[kBlendThreads];  // mx, my, ca, cb
    double2 cc_op[kBlendThreads];
    double4 col[kBlendThreads];
    uint32_t bits[kWarps][kWarps];
};

__global__ void __launch_bounds__(kBlendThreads) k_blend_exact(
    const uint32_t* __restrict__ offsets, const unsigned long long* __restrict__ keys,
    const Gauss64* __restrict__ g64, const Gauss32* __restrict__ g32,
    const GaussCol64* __restrict__ col64, const int width, const int height, const int tiles_x,
    float* __restrict__ image) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BlendSmemExact& s = *reinterpret_cast<BlendSmemExact*>(smem_raw);
    const int tile = blockIdx.x;
    const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = int((warp & 1) * 8 + (lane & 7)), ly = int((warp >> 1) * 4 + (lane >> 3));
    const int x = x0 + lx, y = y0 + ly;
    const bool inside = x < width && y < height;
    const uint32_t b = offsets[tile], e = offsets[tile + 1];
    const double px = double(x) + 0.5, py = double(y) + 0.5;
    double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0;
    bool done = !inside;
    for (uint32_t base = b; base < e; base += kBlendThreads) {
        const uint32_t cnt = min(uint32_t(kBlendThreads), e - base);
        const bool valid = threadIdx.x < cnt;
        unsigned mask = 0;
        if (valid) {
            const uint32_t gi = uint32_t(keys[base + threadIdx.x]);
            const Gauss64 G = g64[gi];
            const GaussCol64 C = col64[gi];
            const double2 m = *reinterpret_cast<const double2*>(&g32[gi].mx);
            s.geo[threadIdx.x] = make_double4(m.x, m.y, G.ca, G.cb);
            s.cc_op[threadIdx.x] = make_double2(G.cc, G.op);
            s.col[threadIdx.x] = make_double4(C.r, C.g, C.b, 0.0);
            const float2 h = *reinterpret_cast<const float2*>(&g32[gi].hx);
            const float mlx = float(m.x - double(x0)), mly = float(m.y - double(y0));
            if (h.x >= 0.0f) {
#pragma unroll
                for (int w = 0; w < kWarps; ++w) {
                    const float bxf = float((w & 1) * 8), byf = float((w >> 1) * 4);
                    const bool hit = mlx - h.x <= bxf + 7.5f && mlx + h.x >= bxf + 0.5f &&
                                     mly - h.y <= byf + 3.5f && mly + h.y >= byf + 0.5f;
                    mask |= hit ? (1u << w) : 0u;
                }
            }
        }
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const unsigned bb = __ballot_sync(0xffffffffu, (mask >> w) & 1u);
            if (lane == 0) s.bits[w][warp] = bb;
        }
        if (__syncthreads_and(done)) break;
        for (int c = 0; c < kWarps; ++c) {
            unsigned bits = s.bits[warp][c];
            while (bits) {
                const int j = c * 32 + (__ffs(bits) - 1);
                bits &= bits - 1;
                if (!done) {
                    const double4 g = s.geo[j];
                    const double2 co = s.cc_op[j];
                    const double alpha = alpha_exact(g.x, g.y, g.z, g.w, co.x, co.y, px, py);
                    if (alpha >= kMinAlpha) {
                        const double4 col = s.col[j];
                        const double w = alpha * T;
                        cr += col.x * w;
                        cg += col.y * w;
                        cb += col.z * w;
                        T *= 1.0 - alpha;
                        done = T < kTermT;
                    }
                }
            }
        }
        __syncthreads();
    }
    if (inside) {
        float* o = image + (size_t(y) * width + x) * 3;
        o[0] = float(cr);
        o[1] = float(cg);
        o[2] = float(cb);
    }
}

// ---------------------------------------------------------------------------
// Exact blend with KPC instrumentation (collect_kpc, rasterizer.hpp:86-96):
// kpc[pair] = sum over the tile's pixels of alpha*T at that pair, accumulated
// exactly as blend_scalar.cpp:16-54 does -- one accumulator per pixel lane
// (x - x0) & 3, each fed in (y, x) scan order, reduced as (a0+a1)+(a2+a3).
// Pixels blend a 32-pair batch and park their weights in shared memory; then
// 128 threads (pair, lane) sum the 4 x 16 weights of their lane in that order.
constexpr int kKpcBatch = 32;

struct KpcSmem {
    double w[kKpcBatch][kTile * kTile];  // per pair, per pixel (row-major) weight
    double part[kKpcBatch][4];
    double4 geo[kKpcBatch];  // mx, my, ca, cb
    double2 cc_op[kKpcBatch];
    double4 col[kKpcBatch];
};

__global__ void __launch_bounds__(kTile * kTile) k_blend_exact_kpc(
    const uint32_t* __restrict__ offsets, const unsigned long long* __restrict__ keys,
    const Gauss64* __restrict__ g64, const Gauss32* __restrict__ g32,
    const GaussCol64* __restrict__ col64, const int width,
    const int height, const int tiles_x, float* __restrict__ image, double* __restrict__ kpc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    KpcSmem& s = *reinterpret_cast<KpcSmem*>(smem_raw);
    const int tile = blockIdx.x;
    const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
    const int lx = int(threadIdx.x & 15), ly = int(threadIdx.x >> 4);
    const int x = x0 + lx, y = y0 + ly;
    const int span_w = min(kTile, width - x0), span_h = min(kTile, height - y0);
    const bool inside = lx < span_w && ly < span_h;
    const uint32_t b = offsets[tile], e = offsets[tile + 1];
    const double px = double(x) + 0.5, py = double(y) + 0.5;
    double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0;
    bool done = !inside;
    for (uint32_t base = b; base < e; base += kKpcBatch) {
        const int cnt = int(min(uint32_t(kKpcBatch), e - base));
        if (int(threadIdx.x) < cnt) {
            const uint32_t gi = uint32_t(keys[base + threadIdx.x]);
            const Gauss64 G = g64[gi];
            const GaussCol64 C = col64[gi];
            const double2 m = *reinterpret_cast<const double2*>(&g32[gi].mx);
            s.geo[threadIdx.x] = make_double4(m.x, m.y, G.ca, G.cb);
            s.cc_op[threadIdx.x] = make_double2(G.cc, G.op);
            s.col[threadIdx.x] = make_double4(C.r, C.g, C.b, 0.0);
        }
        __syncthreads();
        for (int j = 0; j < cnt; ++j) {
            double wj = 0.0;
            if (!done) {
                const double4 g = s.geo[j];
                const double2 co = s.cc_op[j];
                const double alpha = alpha_exact(g.x, g.y, g.z, g.w, co.x, co.y, px, py);
                if (alpha >= kMinAlpha) {
                    const double4 col = s.col[j];
                    wj = alpha * T;
                    cr += col.x * wj;
                    cg += col.y * wj;
                    cb += col.z * wj;
                    T *= 1.0 - alpha;
                    done = T < kTermT;
                }
            }
            s.w[j][threadIdx.x] = wj;
        }
        __syncthreads();
        if (int(threadIdx.x) < 4 * cnt) {
            const int j = int(threadIdx.x) >> 2, lane = int(threadIdx.x) & 3;
            double acc = 0.0;
            for (int yy = 0; yy < span_h; ++yy)
                for (int xx = lane; xx < span_w; xx += 4) acc += s.w[j][yy * kTile + xx];
            s.part[j][lane] = acc;
        }
        __syncthreads();
        if (int(threadIdx.x) < cnt) {
            const int j = int(threadIdx.x);
            kpc[base + j] = (s.part[j][0] + s.part[j][1]) + (s.part[j][2] + s.part[j][3]);
        }
        __syncthreads();
    }
    if (inside) {
        float* o = image + (size_t(y) * width + x) * 3;
        o[0] = float(cr);
        o[1] = float(cg);
        o[2] = float(cb);
    }
}

void launch_blend_exact_kpc(const uint32_t* offsets, const unsigned long long* keys,
                            const Gauss64* g64, const Gauss32* g32, const GaussCol64* col64,
                            int width, int height, int tiles_x, int tiles_y, float* image,
                            double* kpc, cudaStream_t s) {
    const int n_tiles = tiles_x * tiles_y;
    if (n_tiles <= 0) return;
    static bool attr = false;
    const int smem = int(sizeof(KpcSmem));
    if (!attr) {
        cudaFuncSetAttribute(k_blend_exact_kpc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    k_blend_exact_kpc<<<n_tiles, kTile * kTile, smem, s>>>(offsets, keys, g64, g32, col64, width,
                                                           height, tiles_x, image, kpc);
}

// Per-tile GTC (metrics.cpp:18-35): the mean kpc of the tile's pairs, summed
// in sorted order; and one view mean over non-empty tiles in tile order
// (metrics.cpp:37-42) by a single thread, matching the reference's sums.
__global__ void k_tile_gtc(const uint32_t* offsets, int n_tiles, const double* kpc,
                           double* tile_gtc) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    const uint32_t b = offsets[t], e = offsets[t + 1];
    double sum = 0.0;
    for (uint32_t i = b; i < e; ++i) sum += kpc[i];
    tile_gtc[t] = e > b ? sum / double(e - b) : 0.0;
}

__global__ void k_view_gtc(const uint32_t* offsets, int n_tiles, const double* tile_gtc,
                           double* out) {
    double sum = 0.0;
    unsigned long long n = 0;
    for (int t = 0; t < n_tiles; ++t)
        if (offsets[t + 1] > offsets[t]) {
            sum += tile_gtc[t];
            ++n;
        }
    out[0] = n ? sum / double(n) : __longlong_as_double(0x7ff8000000000000ll);
}

// metrics.cpp:44-57: kpc bins [0,0.01) [0.01,0.05) [0.05,0.2) [0.2,1) [1,inf)
__global__ void k_kpc_histogram(const double* kpc, uint64_t n, unsigned long long* bins) {
    __shared__ unsigned long long s[5];
    if (threadIdx.x < 5) s[threadIdx.x] = 0;
    __syncthreads();
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double k = kpc[i];
        const int bin = k < 0.01 ? 0 : k < 0.05 ? 1 : k < 0.2 ? 2 : k < 1.0 ? 3 : 4;
        atomicAdd(&s[bin], 1ull);
    }
    __syncthreads();
    if (threadIdx.x < 5 && s[threadIdx.x]) atomicAdd(&bins[threadIdx.x], s[threadIdx.x]);
}

void launch_view_gtc(const uint32_t* offsets, int n_tiles, const double* kpc, uint64_t n_pairs,
                     double* tile_gtc, double* view_gtc, unsigned long long* bins, cudaStream_t s) {
    if (n_tiles <= 0) return;
    k_tile_gtc<<<(n_tiles + 255) / 256, 256, 0, s>>>(offsets, n_tiles, kpc, tile_gtc);
    k_view_gtc<<<1, 1, 0, s>>>(offsets, n_tiles, tile_gtc, view_gtc);
    if (n_pairs) k_kpc_histogram<<<148, 256, 0, s>>>(kpc, n_pairs, bins);
}

uint64_t blend_record_bytes() { return sizeof(BlendRec); }
int blend_launches() { return 1; }

template <int S>
static void launch_cpa(const uint32_t* offsets, const uint32_t* order,
                       const unsigned long long* keys, const Gauss64* g64, const Gauss32* g32,
                       int width, int height, int tiles_x, int n_tiles, unsigned* ticket,
                       float* image, cudaStream_t s) {
    const int smem = int(sizeof(CpaShared<S>));
    static std::mutex mu;
    static int grid_of[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int grid = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (dev < 0 || dev >= 64 || !grid_of[dev]) {
            cudaFuncSetAttribute(k_blend_cpa<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            int per_sm = 0, n_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_blend_cpa<S>, kCpaThreads, smem);
            cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
            grid = std::max(1, per_sm) * std::max(1, n_sm);
            if (dev >= 0 && dev < 64) grid_of[dev] = grid;
        } else {
            grid = grid_of[dev];
        }
    }
    grid = std::min(n_tiles, grid);
    launch_pdl(k_blend_cpa<S>, grid, kCpaThreads, smem, s, offsets, order, keys, g64, g32, width,
               height, tiles_x, uint32_t(n_tiles), ticket, image);
}

void launch_blend_tiles(const uint32_t* offsets, const uint32_t* order, int n_order,
                        int frame_tiles, const unsigned long long* keys, const Gauss64* g64,
                        const Gauss32* g32, int width, int height, int tiles_x, unsigned* ticket,
                        float* image, cudaStream_t s) {
    if (n_order <= 0) return;
    if (frame_tiles > kCpaBigFrameTiles)
        launch_cpa<kCpaStagesBig>(offsets, order, keys, g64, g32, width, height, tiles_x, n_order,
                                  ticket, image, s);
    else
        launch_cpa<kCpaStages>(offsets, order, keys, g64, g32, width, height, tiles_x, n_order,
                               ticket, image, s);
}

void launch_blend(const uint32_t* offsets, const uint32_t* order, const unsigned long long* keys,
                  const Gauss64* g64, const Gauss32* g32, const GaussCol64* col64, int width,
                  int height, int tiles_x, int tiles_y, bool exact, float* image, cudaStream_t s,
                  unsigned* ticket, void* records, uint64_t n_records, bool records_packed,
                  int kernel) {
    const int n_tiles = tiles_x * tiles_y;
    if (n_tiles <= 0) return;
    if (kernel == kBlendGather4 && !exact && ticket && n_records) {
        CUtensorMap mrow;
        if (encode_row_map(g32, n_records, &mrow)) {
            const int smem = int(sizeof(G4Shared));
            static std::mutex mu;
            static int grid_of[64] = {};
            int dev = 0;
            cudaGetDevice(&dev);
            int grid = 0;
            {
                std::lock_guard<std::mutex> lock(mu);
                if (dev < 0 || dev >= 64 || !grid_of[dev]) {
                    cudaFuncSetAttribute(k_blend_g4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem);
                    int per_sm = 0, n_sm = 0;
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_blend_g4, kG4Threads,
                                                                  smem);
                    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
                    grid = std::max(1, per_sm) * std::max(1, n_sm);
                    if (dev >= 0 && dev < 64) grid_of[dev] = grid;
                } else {
                    grid = grid_of[dev];
                }
            }
            grid = std::min(n_tiles, grid);
            launch_pdl(k_blend_g4, grid, kG4Threads, smem, s, offsets, order, keys, mrow, g64,
                       g32, width, height, tiles_x, uint32_t(n_tiles), ticket, image);
            return;
        }
    }
    if (kernel == kBlendCpa && !exact && ticket) {
        if (n_tiles > kCpaBigFrameTiles)
            launch_cpa<kCpaStagesBig>(offsets, order, keys, g64, g32, width, height, tiles_x,
                                      n_tiles, ticket, image, s);
        else
            launch_cpa<kCpaStages>(offsets, order, keys, g64, g32, width, height, tiles_x,
                                   n_tiles, ticket, image, s);
        return;
    }
    if (kernel == kBlendTma && !exact && records && ticket) {
        BlendRec* rec = static_cast<BlendRec*>(records);
        if (!records_packed)  // the frame's sort writes them; stage entry points pack here
            launch_pdl(k_pack_blend, n_tiles, 128, 0, s, offsets, keys, g64, g32, tiles_x, rec);
        const int smem = int(sizeof(TmaShared));
        static std::mutex mu;
        static int grid_of[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        int grid = 0;
        {
            std::lock_guard<std::mutex> lock(mu);
            if (dev < 0 || dev >= 64 || !grid_of[dev]) {
                cudaFuncSetAttribute(k_blend_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                int per_sm = 0, n_sm = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_blend_tma, kTmaThreads, smem);
                cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
                grid = std::max(1, per_sm) * std::max(1, n_sm);
                if (dev >= 0 && dev < 64) grid_of[dev] = grid;
            } else {
                grid = grid_of[dev];
            }
        }
        grid = std::min(n_tiles, grid);
        launch_pdl(k_blend_tma, grid, kTmaThreads, smem, s, offsets, order,
                   static_cast<const BlendRec*>(rec), g64, g32, width, height, tiles_x,
                   uint32_t(n_tiles), ticket, image);
        return;
    }
    if (exact) {
        static bool attr = false;
        const int smem = int(sizeof(BlendSmemExact));
        if (!attr) {
            cudaFuncSetAttribute(k_blend_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            attr = true;
        }
        k_blend_exact<<<n_tiles, kBlendThreads, smem, s>>>(offsets, keys, g64, g32, col64, width,
                                                            height, tiles_x, image);
    } else {
#ifndef BLEND_WS
#define BLEND_WS 1
#endif
#if BLEND_WS
        const int smem = int(sizeof(WsShared));
        static bool ws_attr[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !ws_attr[dev]) {
            cudaFuncSetAttribute(k_blend_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (dev >= 0 && dev < 64) ws_attr[dev] = true;
        }
#ifndef BLEND_PERSISTENT
#define BLEND_PERSISTENT 1
#endif
#if BLEND_PERSISTENT
        const int smem_p = int(sizeof(WspShared));
        static bool wsp_attr[64] = {};
        static int wsp_grid[64] = {};
        if (dev < 0 || dev >= 64 || !wsp_attr[dev]) {
            cudaFuncSetAttribute(k_blend_wsp, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_p);
            int per_sm = 0, n_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_blend_wsp, kWsThreads, smem_p);
            cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
            if (dev >= 0 && dev < 64) {
                wsp_attr[dev] = true;
                wsp_grid[dev] = std::max(1, per_sm) * std::max(1, n_sm);
            }
        }
        const int grid = std::min(n_tiles, (dev >= 0 && dev < 64) ? wsp_grid[dev] : 444);
        launch_pdl(k_blend_wsp, grid, kWsThreads, smem_p, s, offsets, order, keys, g64, g32, width,
                   height, tiles_x, uint32_t(n_tiles), WSP_DYNAMIC ? ticket : nullptr, image);
        return;
#endif
        launch_pdl(k_blend_ws, n_tiles, kWsThreads, smem, s, offsets, order, keys, g64, g32, width,
                   height, tiles_x, image);
        return;
#endif
        k_blend_fast<<<n_tiles * kFastParts, kFastThreads, 0, s>>>(offsets, order, keys, g64, g32,
                                                                   width, height, tiles_x, image);
    }
}

}  // namespace fgs
