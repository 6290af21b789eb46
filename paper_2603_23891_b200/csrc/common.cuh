// common.cuh -- shared device definitions for the sm_100a FilterGS kernels.
//
// All translation units are compiled with -fmad=false: every FP64 expression
// on the parity path must round exactly like the reference's no-FMA scalar
// code (mark_core.hpp:12-15, proj/CMakeLists.txt:13).  Fast FP32 code that
// wants fused multiply-adds asks for them explicitly with __fmaf_rn.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fgs {

constexpr int kTile = 16;                  // tiles.hpp:8-9
constexpr uint32_t kRootParent = 0xFFFFFFFFu;  // core.hpp:15
constexpr double kAlphaCap = 0.99;         // kernels.hpp:20
constexpr double kMinAlpha = 1.0 / 255.0;  // kernels.hpp:21
constexpr double kTermT = 1e-4;            // kernels.hpp:22

// projection.hpp:23-32 CameraGeom, 44 doubles; passed by value as a kernel
// parameter (352 B, well under the 32 KB parameter limit on sm_100a).
struct Geom {
    double rot[9];
    double trans[3];
    double fx, fy, cx, cy;
    double width, height;
    double znear, zfar;
    double planes[6][4];
};

// Node fields the preprocess gathers for each selected node: one 64-byte
// record so a gather is two 32-byte sectors instead of fourteen SoA sectors.
struct __align__(16) SplatRec {
    float mx, my, mz, sx;
    float sy, sz, qw, qx;
    float qy, qz, opacity, cr;
    float cg, cb, pad0, pad1;
};

// Per projected gaussian, the FP64 conic and opacity (exact blend path, the fast
// blend's guard-band recompute, parity readback); the FP64 mean and radius live in
// the Gauss32 row.  32 bytes.
struct __align__(16) Gauss64 {
    double ca, cb, cc;
    double op;
};
static_assert(sizeof(Gauss64) == 32, "one sector per gaussian");

// FP64 colours, only materialised for the exact (bit-identical) blend.
struct __align__(16) GaussCol64 {
    double r, g, b, pad;
};

// Per projected gaussian, FP32 blend record (48 bytes).
//   e(dx,dy) = ha*dx^2 + cb*dx*dy + hc*dy^2 = -power * log2(e) (coefficients
//   pre-scaled by log2(e)); sample skipped iff e > ethr = log2(255 * opacity)
//   (alpha < 1/255, kernels.hpp:21); alpha = min(op * 2^-e, 0.99).
//   (hx, hy): half-extents of the e <= ethr ellipse, computed in FP64 and
//   rounded outward -- a conservative box outside which the reference
//   provably skips every sample (blend.cu uses it to cull per warp).
//   (mx, my): the FP64 mean (BlendList mean_x/y, bit-exact), so one 64-byte row --
//   two whole 32-byte sectors -- holds everything the fast blend reads for a pair;
//   radius: the FP64 effective radius (BlendList radius; read back only).
struct __align__(16) Gauss32 {
    float ha, cb, hc, ethr;
    float op, r, g, b;
    float hx, hy;
    double radius;
    double mx, my;
};
static_assert(sizeof(Gauss32) == 64, "one 64-byte blend row per gaussian");

// Per projected gaussian, what key duplication needs.
struct __align__(16) GaussEmit {
    uint32_t depth_bits;  // bit_cast<u32>(float(depth)), rasterizer.cpp:113-114
    uint32_t node;
    int16_t tx0, ty0, tx1, ty1;  // inclusive tile rect; tx1 < tx0 => no pairs
};

// Per-kernel device time of the filter (stage timing only): for kernel k, the
// earliest CTA start (stored complemented, so a zeroed slot loses every
// atomicMax) and the latest CTA end, %globaltimer ns.  Kernels: 0-3 the parallel
// filter's F1-F4; serial filter: levels 0..kClockLevels-1, then its compaction.
constexpr int kFilterClocks = 16;
struct FilterClock {
    unsigned long long t0n[kFilterClocks], t1[kFilterClocks];
};

// Device-resident per-frame counters (one cudaMemsetAsync clears them).
struct FrameCounters {
    unsigned long long n_selected;
    unsigned long long n_gaussians;
    unsigned long long n_pairs;
    unsigned int blend_ticket;  // k_blend_wsp's dynamic tile queue
    unsigned int ticket_prep;
    unsigned int ticket_bin;
    unsigned int big_tiles;
    unsigned int overflow;     // pair buffer too small
    unsigned int nonfinite;    // project() produced a non-finite value
    unsigned int big_cursor;
    unsigned int serial_passes;  // filter_serial: levels with an active node
    // OR and OR-of-complement of every reference sort key (tile << 32 | depth bits,
    // rasterizer.cpp:111-115): digit d needs an LSD pass iff it is not uniform
    unsigned long long key_or, key_nand;
    FilterClock clock;  // T_calcu / T_synch split of the filter (stage timing)
};

// Running totals across frames (not cleared per frame).
struct RunTotals {
    unsigned long long frames;
    unsigned long long sum_selected;
    unsigned long long sum_pairs;
    unsigned long long pad;
    // sum over frames of SURVEY 8(d)'s radix-sort bytes (24 B per pair per
    // non-uniform 8-bit digit + 8 B per pair for the histogram)
    unsigned long long sum_sort_bytes;
};

#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// CTAs are dispatched in blockIdx order, so the first start is among the first
// CTAs and the last end among the last ones: only those record (the leaf pass of a
// 50M-node tree has 43K CTAs; one atomic each on one word perturbed the timing).
__device__ __forceinline__ void clock_start(FilterClock* c, int k) {
    if (c && threadIdx.x == 0 && blockIdx.x < 8u) atomicMax(&c->t0n[k], ~global_ns());
}
__device__ __forceinline__ void clock_end(FilterClock* c, int k) {
    if (c && threadIdx.x == 0 && blockIdx.x + 256u >= gridDim.x)
        atomicMax(&c->t1[k], global_ns());
}

// std::max / std::min semantics (first argument NaN propagates), as the
// reference relies on (mark_core.hpp:33,90,110).
__device__ __forceinline__ double std_max(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double std_min(double a, double b) { return (b < a) ? b : a; }

// int(std::floor(x)) with x86 cvttsd2si semantics for out-of-range values
// (INT_MIN), so degenerate inputs bin exactly as the reference binary does.
__device__ __forceinline__ int floor_to_int_x86(double x) {
    const double f = floor(x);
    return (f >= -2147483648.0 && f < 2147483648.0) ? static_cast<int>(f)
                                                     : static_cast<int>(0x80000000u);
}
#endif  // __CUDACC__

}  // namespace fgs
