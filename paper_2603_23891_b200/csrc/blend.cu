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
#include "launch.h"

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

__device__ __forceinline__ void blend_sample_fast(const WarpStage& st, int k, float pxl,
                                                  float pyl, PixState& p, bool& unsure) {
    const float4 geo = st.geo[k];
    const float4 ct = st.ct[k];
    const float2 gb = st.gb[k];
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
    const float t = p.T - w;
    p.T = t < 1e-4f ? 0.0f : t;
}

// The same sample with the reference's FP64 decision wherever the FP32 one is
// uncertain (used only to re-run a batch in which some lane was unsure).
__device__ __forceinline__ void blend_sample_checked(const WarpStage& st, int k, float pxl,
                                                     float pyl, double px, double py,
                                                     const Gauss64* __restrict__ g64,
                                                     PixState& p) {
    const float4 geo = st.geo[k];
    const float4 ct = st.ct[k];
    const float2 gb = st.gb[k];
    const float dx = pxl - geo.x, dy = pyl - geo.y;
    const float Q = __fmaf_rn(geo.z * dx, dx, geo.w * dy * dy);
    const float ev = __fmaf_rn(ct.x * dx, dy, Q);
    const float d = ev - ct.y;
    const float margin = __fmaf_rn(Q, 7.62939453125e-06f, 1.1007e-05f);
    bool take = d < -margin;
    float alpha = fminf(ct.z * ex2_approx(-ev), 0.99f);
    if (fabsf(d) <= margin && p.T > 0.0f) {
        const Gauss64& G = g64[st.gid[k]];
        const double a64 = alpha_exact(G.mx, G.my, G.ca, G.cb, G.cc, G.op, px, py);
        take = a64 >= kMinAlpha;
        alpha = float(a64);
    }
    const float w = take ? alpha * p.T : 0.0f;
    p.cr = __fmaf_rn(ct.w, w, p.cr);
    p.cg = __fmaf_rn(gb.x, w, p.cg);
    p.cb = __fmaf_rn(gb.y, w, p.cb);
    const float t = p.T - w;
    p.T = t < 1e-4f ? 0.0f : t;
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
            r.m = *reinterpret_cast<const double2*>(&g64[gi].mx);
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
            for (int j = 0; j < nh; ++j) blend_sample_checked(st, j, pxl, pyl, px, py, g64, pix);
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
            s.geo[threadIdx.x] = make_double4(G.mx, G.my, G.ca, G.cb);
            s.cc_op[threadIdx.x] = make_double2(G.cc, G.op);
            s.col[threadIdx.x] = make_double4(C.r, C.g, C.b, 0.0);
            const float2 h = *reinterpret_cast<const float2*>(&g32[gi].hx);
            const float mlx = float(G.mx - double(x0)), mly = float(G.my - double(y0));
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
    const Gauss64* __restrict__ g64, const GaussCol64* __restrict__ col64, const int width,
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
            s.geo[threadIdx.x] = make_double4(G.mx, G.my, G.ca, G.cb);
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
                            const Gauss64* g64, const GaussCol64* col64, int width, int height,
                            int tiles_x, int tiles_y, float* image, double* kpc, cudaStream_t s) {
    const int n_tiles = tiles_x * tiles_y;
    if (n_tiles <= 0) return;
    static bool attr = false;
    const int smem = int(sizeof(KpcSmem));
    if (!attr) {
        cudaFuncSetAttribute(k_blend_exact_kpc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    k_blend_exact_kpc<<<n_tiles, kTile * kTile, smem, s>>>(offsets, keys, g64, col64, width, height,
                                                           tiles_x, image, kpc);
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

void launch_blend(const uint32_t* offsets, const uint32_t* order, const unsigned long long* keys,
                  const Gauss64* g64, const Gauss32* g32, const GaussCol64* col64, int width,
                  int height, int tiles_x, int tiles_y, bool exact, float* image, cudaStream_t s) {
    const int n_tiles = tiles_x * tiles_y;
    if (n_tiles <= 0) return;
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
        k_blend_fast<<<n_tiles * kFastParts, kFastThreads, 0, s>>>(offsets, order, keys, g64, g32,
                                                                   width, height, tiles_x, image);
    }
}

}  // namespace fgs
