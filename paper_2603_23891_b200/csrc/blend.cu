// blend.cu -- tile-wise front-to-back alpha blending (K6), reference
// alpha_blend -> blend_scalar (rasterizer.cpp:137-165, blend_scalar.cpp:13-55).
//
// One 256-thread CTA per 16x16 tile, one thread per pixel.  The tile's
// sorted keys are consumed in batches of 256: each thread stages one
// gaussian's record into shared memory, then every pixel walks the batch.
// The CTA stops as soon as every pixel has terminated (__syncthreads_and).
//
// Fast path (default): FP32 per sample, with the reference's FP64 decision
// recomputed exactly whenever the FP32 estimate is within a certified
// margin of the alpha >= 1/255 skip threshold -- a flipped skip would move a
// pixel by up to 1/255 (SURVEY.md section 7 hard part 6), everything else
// is continuous.  The skip test itself needs no exp:
//     alpha = min(op * exp(power), 0.99) < 1/255  <=>  e > ln(255 op),
//     e = -power = ha dx^2 + cb dx dy + hc dy^2 >= 0.
// FP32 error bound: with Q = ha dx^2 + hc dy^2 >= |cb dx dy| (conic is
// positive definite), |e32 - e| <= ~12 ulp * Q, well inside
// margin = (Q + 1) * 2^-17.
//
// Exact path (LODGS_RENDER_EXACT_BLEND): the reference arithmetic in FP64
// with the reference exp_mx (fastexp.hpp:38-50), no FMA: bit-identical
// pixels.
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
__device__ __forceinline__ double alpha_exact(const Gauss64& G, double px, double py) {
    const double dx = px - G.mx;
    const double dy = py - G.my;
    const double t1 = (G.ca * dx) * dx;
    const double t2 = (G.cc * dy) * dy;
    const double t3 = (G.cb * dx) * dy;
    const double power = -0.5 * (t1 + t2) - t3;
    return std_min(G.op * exp_mx(power), kAlphaCap);
}

constexpr int kBlendThreads = 256;

__global__ void __launch_bounds__(kBlendThreads) k_blend_fast(
    const uint32_t* __restrict__ offsets, const unsigned long long* __restrict__ keys,
    const Gauss64* __restrict__ g64, const Gauss32* __restrict__ g32, const int width,
    const int height, const int tiles_x, float* __restrict__ image) {
    __shared__ float4 s_geo[kBlendThreads];  // mlx, mly, ha, hc
    __shared__ float2 s_ct[kBlendThreads];   // cb, ethr
    __shared__ float4 s_col[kBlendThreads];  // op, r, g, b
    __shared__ uint32_t s_gid[kBlendThreads];

    const int tile = blockIdx.x;
    const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int x = x0 + lx, y = y0 + ly;
    const bool inside = x < width && y < height;
    const uint32_t b = offsets[tile], e = offsets[tile + 1];

    const float pxl = float(lx) + 0.5f, pyl = float(ly) + 0.5f;
    const double px = double(x) + 0.5, py = double(y) + 0.5;
    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
    bool done = !inside;

    for (uint32_t base = b; base < e; base += kBlendThreads) {
        const int cnt = int(min(uint32_t(kBlendThreads), e - base));
        if (int(threadIdx.x) < cnt) {
            const uint32_t gi = uint32_t(keys[base + threadIdx.x]);
            const double2 m = *reinterpret_cast<const double2*>(&g64[gi].mx);
            const float4 q0 = *reinterpret_cast<const float4*>(&g32[gi].ha);
            const float4 q1 = *reinterpret_cast<const float4*>(&g32[gi].op);
            s_geo[threadIdx.x] = make_float4(float(m.x - double(x0)), float(m.y - double(y0)), q0.x, q0.z);
            s_ct[threadIdx.x] = make_float2(q0.y, q0.w);
            s_col[threadIdx.x] = q1;
            s_gid[threadIdx.x] = gi;
        }
        if (__syncthreads_and(done)) break;
        if (!done) {
            for (int j = 0; j < cnt; ++j) {
                const float4 geo = s_geo[j];
                const float2 ct = s_ct[j];
                const float dx = pxl - geo.x, dy = pyl - geo.y;
                const float Q = __fmaf_rn(geo.z * dx, dx, geo.w * dy * dy);
                const float ev = __fmaf_rn(ct.x * dx, dy, Q);
                const float d = ev - ct.y;
                const float margin = __fmaf_rn(Q, 7.62939453125e-06f, 7.62939453125e-06f);
                if (d > margin) continue;  // alpha < 1/255 for certain
                const float4 col = s_col[j];
                float alpha;
                if (d < -margin) {
                    alpha = fminf(col.x * __expf(-ev), 0.99f);
                } else {
                    const double a64 = alpha_exact(g64[s_gid[j]], px, py);
                    if (a64 < kMinAlpha) continue;
                    alpha = float(a64);
                }
                const float w = alpha * T;
                cr = __fmaf_rn(col.y, w, cr);
                cg = __fmaf_rn(col.z, w, cg);
                cb = __fmaf_rn(col.w, w, cb);
                T = T * (1.0f - alpha);
                if (T < 1e-4f) {
                    done = true;
                    break;
                }
            }
        }
        __syncthreads();
    }
    if (inside) {
        float* o = image + (size_t(y) * width + x) * 3;
        o[0] = cr;
        o[1] = cg;
        o[2] = cb;
    }
}

__global__ void __launch_bounds__(kBlendThreads) k_blend_exact(
    const uint32_t* __restrict__ offsets, const unsigned long long* __restrict__ keys,
    const Gauss64* __restrict__ g64, const GaussCol64* __restrict__ col64, const int width,
    const int height, const int tiles_x, float* __restrict__ image) {
    __shared__ Gauss64 s_g[kBlendThreads];
    __shared__ GaussCol64 s_c[kBlendThreads];
    const int tile = blockIdx.x;
    const int x0 = (tile % tiles_x) * kTile, y0 = (tile / tiles_x) * kTile;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int x = x0 + lx, y = y0 + ly;
    const bool inside = x < width && y < height;
    const uint32_t b = offsets[tile], e = offsets[tile + 1];
    const double px = double(x) + 0.5, py = double(y) + 0.5;
    double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0;
    bool done = !inside;
    for (uint32_t base = b; base < e; base += kBlendThreads) {
        const int cnt = int(min(uint32_t(kBlendThreads), e - base));
        if (int(threadIdx.x) < cnt) {
            const uint32_t gi = uint32_t(keys[base + threadIdx.x]);
            s_g[threadIdx.x] = g64[gi];
            s_c[threadIdx.x] = col64[gi];
        }
        if (__syncthreads_and(done)) break;
        if (!done) {
            for (int j = 0; j < cnt; ++j) {
                const double alpha = alpha_exact(s_g[j], px, py);
                if (alpha < kMinAlpha) continue;
                const double w = alpha * T;
                cr += s_c[j].r * w;
                cg += s_c[j].g * w;
                cb += s_c[j].b * w;
                T *= 1.0 - alpha;
                if (T < kTermT) {
                    done = true;
                    break;
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
    if (exact)
        k_blend_exact<<<n_tiles, kBlendThreads, 0, s>>>(offsets, keys, g64, col64, width, height,
                                                        tiles_x, image);
    else
        k_blend_fast<<<n_tiles, kBlendThreads, 0, s>>>(offsets, keys, g64, g32, width, height,
                                                       tiles_x, image);
}

}  // namespace fgs
