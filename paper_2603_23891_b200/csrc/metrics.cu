// metrics.cu -- image metrics and 8-bit output on the device (SURVEY.md 8(f)
// row 4): the reference's psnr / ssim (metrics.cpp:121-195) and save_ppm's
// quantisation (image.cpp:12-28), so per-frame quality checks need no
// float-image round trip to the host.
//
// Determinism: every partial sum has a fixed shape (per-CTA tree, then one
// CTA summing the partials in index order), so a metric is bit-reproducible
// run to run.  It is not bit-equal to the reference's strictly sequential
// double sums (different association); SSIM's per-window value is computed
// with the reference's exact operation order (-fmad=false), only the sum
// over windows is re-associated.
#include "launch.h"

namespace fgs {

constexpr int kMetricThreads = 256;

// image.cpp:19-22: v = clamp(v, 0, 1); byte = uint8(floor(v * 255.f + 0.5f))
__global__ void k_rgb8(const float* __restrict__ img, uint64_t n, uint8_t* __restrict__ out) {
    const uint64_t i0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (i0 + 4 <= n) {
        const float4 v = *reinterpret_cast<const float4*>(img + i0);
        const float a[4] = {v.x, v.y, v.z, v.w};
        uchar4 o;
        unsigned char* b = reinterpret_cast<unsigned char*>(&o);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float x = a[k];
            x = x < 0.f ? 0.f : (x > 1.f ? 1.f : x);
            b[k] = uint8_t(floorf(x * 255.f + 0.5f));
        }
        *reinterpret_cast<uchar4*>(out + i0) = o;
    } else {
        for (uint64_t i = i0; i < n; ++i) {
            float x = img[i];
            x = x < 0.f ? 0.f : (x > 1.f ? 1.f : x);
            out[i] = uint8_t(floorf(x * 255.f + 0.5f));
        }
    }
}

__device__ __forceinline__ double block_sum(double v, double* s_red) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kMetricThreads / 32; ++w) t += s_red[w];
    return t;
}

// metrics.cpp:121-132: sum over channels of (double(a) - double(b))^2, one
// contiguous chunk per CTA.
__global__ void __launch_bounds__(kMetricThreads) k_sq_diff(const float* __restrict__ a,
                                                            const float* __restrict__ b,
                                                            uint64_t n, uint64_t chunk,
                                                            double* __restrict__ partial) {
    __shared__ double s_red[kMetricThreads / 32];
    const uint64_t lo = uint64_t(blockIdx.x) * chunk, hi = lo + chunk < n ? lo + chunk : n;
    double se = 0.0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += kMetricThreads) {
        const double d = double(a[i]) - double(b[i]);
        se += d * d;
    }
    const double t = block_sum(se, s_red);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// metrics.cpp:136-192: one 11x11 window (channel c, origin x0, y0) per thread,
// the reference's per-tap accumulation order; windows ordered (c, y0, x0).
struct SsimWeights {
    double w[121];
};

__global__ void __launch_bounds__(kMetricThreads) k_ssim(const float* __restrict__ a,
                                                         const float* __restrict__ b, int width,
                                                         int height, uint64_t chunk,
                                                         const __grid_constant__ SsimWeights win,
                                                         double* __restrict__ partial) {
    __shared__ double s_red[kMetricThreads / 32];
    constexpr int W = 11;
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    const uint64_t wx = uint64_t(width - W + 1), wy = uint64_t(height - W + 1);
    const uint64_t n_win = 3 * wx * wy;
    const uint64_t lo = uint64_t(blockIdx.x) * chunk, hi = lo + chunk < n_win ? lo + chunk : n_win;
    double total = 0.0;
    for (uint64_t k = lo + threadIdx.x; k < hi; k += kMetricThreads) {
        const int c = int(k / (wx * wy));
        const uint64_t r = k - uint64_t(c) * wx * wy;
        const int y0 = int(r / wx), x0 = int(r - uint64_t(y0) * wx);
        double sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
        for (int dy = 0; dy < W; ++dy) {
            const uint64_t row = (uint64_t(y0 + dy) * uint64_t(width) + uint64_t(x0)) * 3 + c;
#pragma unroll
            for (int dx = 0; dx < W; ++dx) {
                const double wgt = win.w[dy * W + dx];
                const double pa = __ldg(a + row + uint64_t(dx) * 3);
                const double pb = __ldg(b + row + uint64_t(dx) * 3);
                sx += wgt * pa;
                sy += wgt * pb;
                sxx += wgt * pa * pa;
                syy += wgt * pb * pb;
                sxy += wgt * (pa * pb);
            }
        }
        const double vx = sxx - sx * sx, vy = syy - sy * sy;
        const double cov = sxy - sx * sy;
        total += ((2.0 * sx * sy + c1) * (2.0 * cov + c2)) /
                 ((sx * sx + sy * sy + c1) * (vx + vy + c2));
    }
    const double t = block_sum(total, s_red);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// Sums `m` partials in index order (one thread: m <= a few thousand).
__global__ void k_sum_ordered(const double* __restrict__ partial, int m, double* out) {
    if (threadIdx.x != 0) return;
    double t = 0.0;
    for (int i = 0; i < m; ++i) t += partial[i];
    *out = t;
}

void launch_rgb8(const float* img, uint64_t n, uint8_t* out, cudaStream_t s) {
    if (n == 0) return;
    const uint64_t threads = (n + 3) / 4;
    k_rgb8<<<unsigned((threads + 255) / 256), 256, 0, s>>>(img, n, out);
}

// Sum of squared differences; `partial` needs kMetricParts doubles + 1.
void launch_sq_diff(const float* a, const float* b, uint64_t n, double* partial, double* out,
                    cudaStream_t s) {
    const uint64_t chunk = (n + kMetricParts - 1) / kMetricParts;
    const unsigned grid = unsigned(chunk ? (n + chunk - 1) / chunk : 1);
    k_sq_diff<<<grid, kMetricThreads, 0, s>>>(a, b, n, chunk ? chunk : 1, partial);
    k_sum_ordered<<<1, 32, 0, s>>>(partial, int(grid), out);
}

void launch_ssim(const float* a, const float* b, int width, int height, const double* weights,
                 double* partial, double* out, cudaStream_t s) {
    SsimWeights w;
    for (int i = 0; i < 121; ++i) w.w[i] = weights[i];
    const uint64_t n_win = 3ull * uint64_t(width - 10) * uint64_t(height - 10);
    const uint64_t chunk = (n_win + kMetricParts - 1) / kMetricParts;
    const unsigned grid = unsigned((n_win + chunk - 1) / chunk);
    k_ssim<<<grid, kMetricThreads, 0, s>>>(a, b, width, height, chunk, w, partial);
    k_sum_ordered<<<1, 32, 0, s>>>(partial, int(grid), out);
}

}  // namespace fgs
