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

// A hit splat, expanded around the centre of the warp's 8x4 block:
//   e'(x, y) = A x^2 + B xy + C y^2 + D x + E y + F = e - ln(255 op),
// (x, y) = pixel centre minus block centre, so x in [-3.5, 3.5], y in [-1.5, 1.5].
// alpha = op exp(-e) = exp(-e') / 255; the reference skips iff e' > 0.
struct WarpStage {
    float4 c0[32];   // A, B, C, D
    float4 c1[32];   // E, F, M (certified |e'32 - e'| bound over the block), gid bits
    float4 col[32];  // r, g, b, -
};

// Coefficients and the error bound M for one splat relative to block centre (u, v).
// Every FP32 rounding in forming D, E, F and in the five-FMA evaluation is at
// most 2^-24 of a magnitude that S below dominates term by term (the quadratic
// and linear parts at |x| <= 3.5, |y| <= 1.5, the expansion of F, and ethr);
// with the FP32 conic itself off by 2^-24 relative, |e'32 - e'| <= 2^-21 S.
// M = 2^-20 S leaves a further factor of two.
__device__ __forceinline__ void expand_splat(float u, float v, float ha, float cb, float hc,
                                             float ethr, float4& c0, float4& c1,
                                             uint32_t gid) {
    const float hu = ha * u, hv = hc * v, bu = cb * u, bv = cb * v;
    const float D = -__fmaf_rn(2.0f, hu, bv);
    const float E = -__fmaf_rn(2.0f, hv, bu);
    const float quad = __fmaf_rn(hu, u, __fmaf_rn(bu, v, hv * v));
    const float F = quad - ethr;
    const float S = ha * 12.25f + fabsf(cb) * 5.25f + hc * 2.25f +
                    (fabsf(D) + 2.0f * fabsf(hu) + fabsf(bv)) * 3.5f +
                    (fabsf(E) + fabsf(bu) + 2.0f * fabsf(hv)) * 1.5f + fabsf(F) +
                    fabsf(hu * u) + fabsf(bu * v) + fabsf(hv * v) + fabsf(ethr);
    c0 = make_float4(ha, cb, hc, D);
    c1 = make_float4(E, F, S * 9.5367431640625e-07f + 1e-30f, __uint_as_float(gid));
}

// One splat's blend inputs as copied by cp.async (4 x 16 B).
struct __align__(16) RecSlot {
    double2 m;   // mean x, y (Gauss64)
    float4 q0;   // ha, cb, hc, ethr
    float4 col;  // op, r, g, b
    float4 h;    // hx, hy, pad, pad
};
struct RecBuf {
    RecSlot s[32];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(kFastThreads, 10) k_blend_fast(
    const uint32_t* __restrict__ offsets, const unsigned long long* __restrict__ keys,
    const Gauss64* __restrict__ g64, const Gauss32* __restrict__ g32, const int width,
    const int height, const int tiles_x, float* __restrict__ image) {
    __shared__ WarpStage stage[kFastWarps];
    __shared__ __align__(16) RecBuf recs[kFastWarps][2];
    const int tile = blockIdx.x / kFastParts, part = blockIdx.x % kFastParts;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpStage& st = stage[warp];
    // this warp's 8x4 block origin in image pixels
    const int bx = (tile % tiles_x) * kTile + int(warp & 1) * 8;
    const int by = (tile / tiles_x) * kTile + part * 8 + int(warp >> 1) * 4;
    const int x = bx + int(lane & 7), y = by + int(lane >> 3);
    const bool inside = x < width && y < height;
    const uint32_t b = offsets[tile], e = offsets[tile + 1];

    // pixel centre relative to the block centre (bx + 4, by + 2); exact in FP32
    const float qx = float(lane & 7) - 3.5f, qy = float(lane >> 3) - 1.5f;
    const double px = double(x) + 0.5, py = double(y) + 0.5;
    const double cx = double(bx) + 4.0, cy = double(by) + 2.0;
    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
    bool done = !inside;
    if (__all_sync(0xffffffffu, done)) return;

    // Pipeline over 32-splat batches: each lane cp.async-copies the record of
    // "its" splat of the next batch into the warp's shared buffer while the
    // current batch is blended; keys are fetched two batches ahead.  Only the
    // copying lane reads a slot, so per-thread wait_group suffices.
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    auto load_key = [&](uint32_t at) -> uint32_t {
        return at + lane < e ? uint32_t(keys[at + lane]) : kNone;
    };
    auto fetch = [&](uint32_t gi, int buf) {
        if (gi != kNone) {
            RecSlot& d = recs[warp][buf].s[lane];
            cp_async16(&d.m, &g64[gi].mx);
            cp_async16(&d.q0, &g32[gi].ha);
            cp_async16(&d.col, &g32[gi].op);
            cp_async16(&d.h, &g32[gi].hx);
        }
        cp_async_commit();
    };
    uint32_t gi_cur = load_key(b), gi_next = load_key(b + 32);
    fetch(gi_cur, 0);
    int buf = 0;
    for (uint32_t base = b; base < e; base += 32, buf ^= 1) {
        fetch(gi_next, buf ^ 1);
        const uint32_t gi_after = load_key(base + 64);
        cp_async_wait<1>();  // this lane's record of the current batch has landed
        // ---- stage the splats of this batch that touch this warp's block
        bool hit = false;
        if (gi_cur != kNone) {
            const RecSlot& r = recs[warp][buf].s[lane];
            const double2 m = r.m;
            const float4 h4 = r.h;
            const float u = float(m.x - cx), v = float(m.y - cy);
            // pixel centres of the block span [-3.5, 3.5] x [-1.5, 1.5]
            hit = h4.x >= 0.0f && u - h4.x <= 3.5f && u + h4.x >= -3.5f && v - h4.y <= 1.5f &&
                  v + h4.y >= -1.5f;
            if (hit) {
                const float4 q0 = r.q0, col = r.col;
                float4 c0, c1;
                expand_splat(u, v, q0.x, q0.y, q0.z, q0.w, c0, c1, gi_cur);
                st.c0[lane] = c0;
                st.c1[lane] = c1;
                st.col[lane] = make_float4(col.y, col.z, col.w, 0.0f);
            }
        }
        unsigned bits = __ballot_sync(0xffffffffu, hit);
        __syncwarp();
        // ---- blend them front to back
        const float qxx = qx * qx, qxy = qx * qy, qyy = qy * qy;
        while (bits) {
            const int j = __ffs(bits) - 1;
            bits &= bits - 1;
            const float4 c0 = st.c0[j];
            const float4 c1 = st.c1[j];
            const float4 col = st.col[j];
            const float ep = __fmaf_rn(c0.x, qxx, __fmaf_rn(c0.y, qxy, __fmaf_rn(c0.z, qyy,
                             __fmaf_rn(c0.w, qx, __fmaf_rn(c1.x, qy, c1.y)))));
            const float M = c1.z;
            // alpha = exp(-e') / 255 = 2^(-e' log2(e) - log2(255))
            float alpha = fminf(ex2_approx(__fmaf_rn(ep, -1.4426950408889634f, -7.9943534368588578f)),
                                0.99f);
            bool take = ep < -M;
            const bool unsure = !done && fabsf(ep) <= M;
            if (__any_sync(0xffffffffu, unsure)) {  // rare: certified FP64 decision
                if (unsure) {
                    const Gauss64& G = g64[__float_as_uint(c1.w)];
                    const double a64 = alpha_exact(G.mx, G.my, G.ca, G.cb, G.cc, G.op, px, py);
                    take = a64 >= kMinAlpha;
                    alpha = float(a64);
                }
            }
            const float w = (take && !done) ? alpha * T : 0.0f;
            cr = __fmaf_rn(col.x, w, cr);
            cg = __fmaf_rn(col.y, w, cg);
            cb = __fmaf_rn(col.z, w, cb);
            T = T - w;
            done = done || T < 1e-4f;
        }
        if (__all_sync(0xffffffffu, done)) break;
        __syncwarp();
        gi_cur = gi_next;
        gi_next = gi_after;
    }
    cp_async_wait<0>();
    if (inside) {
        float* o = image + (size_t(y) * width + x) * 3;
        o[0] = cr;
        o[1] = cg;
        o[2] = cb;
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

void launch_blend(const uint32_t* offsets, const unsigned long long* keys, const Gauss64* g64,
                  const Gauss32* g32, const GaussCol64* col64, int width, int height,
                  int tiles_x, int tiles_y, bool exact, float* image, cudaStream_t s) {
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
        k_blend_fast<<<n_tiles * kFastParts, kFastThreads, 0, s>>>(offsets, keys, g64, g32, width,
                                                                   height, tiles_x, image);
    }
}

}  // namespace fgs
