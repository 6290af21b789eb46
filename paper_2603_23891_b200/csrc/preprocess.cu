// preprocess.cu -- projection + GTC shrink + tile rect (K3) and Gaussian-tile
// key duplication (K4).
//
// K3 restates prepare_gaussians (rasterizer.cpp:48-73): project() per
// selected node (projection.cpp:60-91, mark_core with tau_r = inf), drop the
// ones short of the near plane, effective_radius (rasterizer.cpp:36-46) and
// the 16x16 tile rect of bin_to_tiles (rasterizer.cpp:78-91).  All FP64,
// exact.  Survivors are compacted in selected order by a chained scan, so a
// gaussian's index is exactly its BlendList position in the reference.  Each
// survivor bumps the pair count of every tile it overlaps (L2 atomics).
//
// K4 scatters one key per (gaussian, tile) straight into its tile's bucket:
// the first radix digit of the (tile, depth) sort is done here by counting.
// key = bit_cast<u32>(depth) << 32 | gaussian; the in-tile order is settled
// by sort.cu, and since gaussian indices are unique per tile the final
// order equals the reference's stable LSD radix (rasterizer.cpp:100-135).
#include <cooperative_groups.h>

#include "launch.h"
#include "pdl.cuh"
#include "mark.cuh"
#include "scan.cuh"

namespace fgs {

// rasterizer.cpp:36-46 (kind 0 three_sigma, 1 fixed, 2 adaptive; tau
// already validated on the host).  log() is CUDA's (<= 1 ulp); the parity
// tests count radius / tile-rect mismatches against glibc.
__device__ __forceinline__ double effective_radius(double sigma_max, float opacity, int kind,
                                                   double tau) {
    const double three_sigma = 3.0 * sigma_max;
    if (kind == 0) return three_sigma;
    const double a0 = double(opacity);
    if (a0 <= tau) return 0.0;
    const double r = sigma_max * sqrt(2.0 * log(a0 / tau));
    return std_min(r, three_sigma);
}

struct Projected {
    bool keep;
    bool nonfinite;
    double mx, my, ca, cb, cc, radius, depth;
};

// projection.cpp:60-91 + effective_radius, with mark_core's world covariance
// from sigma3d (mark.cuh, mark_core.hpp's operations).  known_visible:
// the node passed this frame's filter, whose frustum decision is the same
// FP64 decision (mark_core.hpp:32-40), so the test is not repeated.
__device__ __forceinline__ Projected project_one(const Geom& g, const SplatRec& r,
                                                 const Sigma3& S, int kind, double tau,
                                                 bool known_visible) {
    Projected p;
    p.keep = false;
    p.nonfinite = false;
    MarkOut m;
    cam_transform(g, r.mx, r.my, r.mz, m.tx, m.ty, m.tz);
    if (!known_visible) {
        const double smax = std_max(std_max(double(r.sx), double(r.sy)), double(r.sz));
        if (!frustum_literal(g, m.tx, m.ty, m.tz, 3.0 * smax)) return p;
    }
    if (!(m.tz >= g.znear)) return p;  // z_ok (mark_core.hpp:41)
    ewa_from_sigma<false>(g, m.tx, m.ty, m.tz, S, m);
    // projection.cpp:73 divides by tz; ewa used 1 / max(tz, 1e-12), the same
    // quotient whenever tz >= 1e-12
    const double inv_z = m.tz < 1e-12 ? 1.0 / m.tz : m.inv_zc;
    p.mx = g.fx * (m.tx * inv_z) + g.cx;
    p.my = g.fy * (m.ty * inv_z) + g.cy;
    const double det = m.a * m.c - m.b * m.b;
    p.ca = m.c / det;
    p.cb = -m.b / det;
    p.cc = m.a / det;
    const double sigma_max = sqrt(m.lambda_max);
    p.depth = m.tz;
    // projection.cpp:85-89 checks sigma_min = sqrt(lambda_min) and mark_core's
    // radius = 3 sqrt(lambda_max) for finiteness: for a finite argument x,
    // sqrt(x) is finite iff x >= 0 (NaN otherwise; sqrt(-0) = -0), and 3 sigma_max
    // is finite iff sigma_max is -- the same predicate without the two roots.
    const bool sigma_min_finite = isfinite(m.lambda_min) && m.lambda_min >= 0.0;
    p.nonfinite = !(isfinite(p.mx) && isfinite(p.my) && isfinite(m.a) && isfinite(m.b) &&
                    isfinite(m.c) && isfinite(p.ca) && isfinite(p.cb) && isfinite(p.cc) &&
                    isfinite(sigma_max) && sigma_min_finite && isfinite(m.tz));
    p.radius = effective_radius(sigma_max, r.opacity, kind, tau);
    p.keep = true;
    return p;
}

__device__ __forceinline__ void tile_rect(double mx, double my, double r, int tiles_x,
                                          int tiles_y, GaussEmit& e) {
    if (!(r > 0.0)) {
        e.tx0 = 0;
        e.tx1 = -1;
        e.ty0 = 0;
        e.ty1 = -1;
        return;
    }
    int tx0 = floor_to_int_x86((mx - r) / kTile);
    int tx1 = floor_to_int_x86((mx + r) / kTile);
    int ty0 = floor_to_int_x86((my - r) / kTile);
    int ty1 = floor_to_int_x86((my + r) / kTile);
    tx0 = max(tx0, 0);
    ty0 = max(ty0, 0);
    tx1 = min(tx1, tiles_x - 1);
    ty1 = min(ty1, tiles_y - 1);
    if (tx1 < tx0 || ty1 < ty0) {
        tx0 = 0;
        tx1 = -1;
        ty0 = 0;
        ty1 = -1;
    }
    e.tx0 = int16_t(tx0);
    e.tx1 = int16_t(tx1);
    e.ty0 = int16_t(ty0);
    e.ty1 = int16_t(ty1);
}

__device__ __forceinline__ uint32_t rect_count(const GaussEmit& e) {
    return (e.tx1 < e.tx0) ? 0u : uint32_t(e.tx1 - e.tx0 + 1) * uint32_t(e.ty1 - e.ty0 + 1);
}

#ifndef PREP_FP64_THR
#define PREP_FP64_THR 0
#endif
// FP32 blend record from the FP64 gaussian (blend.cu explains ethr).
__device__ __forceinline__ Gauss32 make_g32(double ca, double cb, double cc, double op, double r,
                                            double gg, double b, double mx, double my,
                                            double radius) {
    Gauss32 o;
    o.mx = mx;
    o.my = my;
    o.radius = radius;
    // exponent coefficients pre-scaled by log2(e): the blend evaluates
    // e' = e log2(e) and alpha = op * 2^-e' with one MUFU.EX2
    constexpr double kLog2e = 1.4426950408889634074;
    o.ha = float(0.5 * ca * kLog2e);
    o.cb = float(cb * kLog2e);
    o.hc = float(0.5 * cc * kLog2e);
    // The skip threshold in FP32, log2f(255 op) (<= 1 ulp; 255 op rounds once): the
    // blend's certified margin carries a constant log2(e) 2^-17 = 1.1e-5 for the
    // threshold's rounding, 20x the error here, so every FP32 decision it trusts is
    // still the reference's.  (An FP64 log here was ~5 % of the kernel's issue.)
#if PREP_FP64_THR  // experiment: the FP64 threshold and box of round 1
    const double ethr64 = log(255.0 * op);
    const float ethr2 = float(ethr64 * kLog2e);
#else
    const float ethr2 = log2f(255.0f * float(op));
#endif
    o.ethr = ethr2;
    o.op = float(op);
    o.r = float(r);
    o.g = float(gg);
    o.b = float(b);
    // Box of the ellipse e <= E, E the threshold inflated past every rounding of
    // the FP32 threshold above and of the reference's own alpha test (exp_mx is
    // within 1e-15 of exp): for the quadratic form [[ha, cb/2], [cb/2, hc]],
    // |dx| <= sqrt(E hc / det) and |dy| <= sqrt(E ha / det).  det in FP64 (the
    // cancellation), the rest in FP32 with directed rounding (inputs rounded up,
    // det down, every operation rounded up), then 1e-3 px for the FP32 tile-local
    // mean.  E <= 0 (opacity <= 1/255): nothing ever blends.
    const double ethr = double(ethr2) * 0.69314718055994530942;
    const double E = ethr + 1e-5 * (1.0 + fabs(ethr));
    const double ha = 0.5 * ca, hc = 0.5 * cc;
    const double det = ha * hc - 0.25 * cb * cb;
    const float detf = __double2float_rd(det * (1.0 - 1e-9));
    if (E > 0.0 && detf > 0.0f) {
        const float Ef = __double2float_ru(E);
        const float qx = __fdiv_ru(__fmul_ru(Ef, __double2float_ru(hc)), detf);
        const float qy = __fdiv_ru(__fmul_ru(Ef, __double2float_ru(ha)), detf);
        o.hx = __fadd_ru(__fsqrt_ru(qx), 1e-3f);
        o.hy = __fadd_ru(__fsqrt_ru(qy), 1e-3f);
    } else if (E > 0.0) {  // degenerate or tiny det: never cull
        o.hx = o.hy = 3.0e38f;
    } else {
        o.hx = o.hy = -1.0f;
    }
    return o;
}

// Contiguous slice [lo, hi) of n items for this CTA (keeps a CTA's splats
// spatially coherent, so its shared-memory tile histogram stays sparse).
__device__ __forceinline__ void cta_range(uint64_t n, uint64_t& lo, uint64_t& hi) {
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    lo = min(n, uint64_t(blockIdx.x) * per);
    hi = min(n, lo + per);
}

// Block-wide sum of two counters, added once to global memory.
__device__ __forceinline__ void block_add2(uint32_t a, uint32_t b, unsigned long long* ga,
                                           unsigned long long* gb) {
    __shared__ unsigned long long s_sum[2];
    if (threadIdx.x == 0) s_sum[0] = s_sum[1] = 0;
    __syncthreads();
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, off);
        b += __shfl_down_sync(0xffffffffu, b, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (a) atomicAdd(&s_sum[0], (unsigned long long)a);
        if (b) atomicAdd(&s_sum[1], (unsigned long long)b);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_sum[0]) atomicAdd(ga, s_sum[0]);
        if (s_sum[1]) atomicAdd(gb, s_sum[1]);
    }
}

// Records are indexed by selected slot s; a slot whose node fails projection
// (rasterizer.cpp:56, near-plane drop) gets an empty rect tagged kDropped.
// Keys carry the slot, whose order equals BlendList order, so the sort is
// unchanged; the slot -> BlendList index map is only built for readbacks.
#ifndef PREP_MIN_CTAS
#define PREP_MIN_CTAS 4
#endif
__global__ void __launch_bounds__(kPrepBlock, PREP_MIN_CTAS) k_preprocess(
    const Geom g, const SplatRec* __restrict__ splat, const uint32_t* __restrict__ selected, const int kind, const double tau, const int tiles_x,
    const int tiles_y, PrepOut out, FrameCounters* cnt, const int use_hist,
    const int known_visible) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    extern __shared__ uint32_t s_hist[];
    const int n_tiles = tiles_x * tiles_y;
    uint64_t lo, hi;
    cta_range(cnt->n_selected, lo, hi);
    if (use_hist)
        for (int t = threadIdx.x; t < n_tiles; t += kPrepBlock) s_hist[t] = 0u;
    __syncthreads();
    uint32_t kept = 0, pairs = 0;
    unsigned long long kor = 0, knand = 0;
    // The next slot's index is in flight while this one is projected (a deeper
    // prefetch of the 64-byte record spilled at 64 registers and was slower).
    // The world covariance is recomputed from the record (sigma3d, the same FP64
    // operations as mark_core) rather than read: 48 B per node less HBM traffic
    // and storage, for ~200 FP64 instructions the kernel had issue room for.
    uint64_t s = lo + threadIdx.x;
    uint32_t idx_next = s < hi ? __ldg(selected + s) : 0u;
#ifndef PREP_L2PF
#define PREP_L2PF 1
#endif
#if PREP_L2PF
    // the slot after next's index, and the next slot's record pulled into L2
    // (no registers held): its load then waits on L2, not HBM
    uint32_t idx_after = s + kPrepBlock < hi ? __ldg(selected + s + kPrepBlock) : 0u;
#endif
    for (; s < hi; s += kPrepBlock) {
        const uint32_t idx = idx_next;
#if PREP_L2PF
        idx_next = idx_after;
        if (s + kPrepBlock < hi)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(splat + idx_next));
        if (s + 2 * kPrepBlock < hi) idx_after = __ldg(selected + s + 2 * kPrepBlock);
#else
        if (s + kPrepBlock < hi) idx_next = __ldg(selected + s + kPrepBlock);
#endif
        const float4* src = reinterpret_cast<const float4*>(splat + idx);
        const float4 a = __ldg(src), b = __ldg(src + 1), c = __ldg(src + 2), d = __ldg(src + 3);
        SplatRec rec;
        rec.mx = a.x; rec.my = a.y; rec.mz = a.z; rec.sx = a.w;
        rec.sy = b.x; rec.sz = b.y; rec.qw = b.z; rec.qx = b.w;
        rec.qy = c.x; rec.qz = c.y; rec.opacity = c.z; rec.cr = c.w;
        rec.cg = d.x; rec.cb = d.y;
        const Sigma3 S = sigma3d(rec.sx, rec.sy, rec.sz, rec.qw, rec.qx, rec.qy, rec.qz);
        const Projected p = project_one(g, rec, S, kind, tau, known_visible != 0);
        GaussEmit e;
        e.node = idx;
        if (p.keep) {
            if (p.nonfinite) atomicOr(&cnt->nonfinite, 1u);
            Gauss64 r64;
            r64.ca = p.ca;
            r64.cb = p.cb;
            r64.cc = p.cc;
            r64.op = double(rec.opacity);
            out.g64[s] = r64;
            if (out.col64) {
                GaussCol64 col;
                col.r = double(rec.cr);
                col.g = double(rec.cg);
                col.b = double(rec.cb);
                col.pad = 0.0;
                out.col64[s] = col;
            }
            out.g32[s] = make_g32(p.ca, p.cb, p.cc, double(rec.opacity), double(rec.cr),
                                  double(rec.cg), double(rec.cb), p.mx, p.my, p.radius);
            e.depth_bits = __float_as_uint(__double2float_rn(p.depth));
            tile_rect(p.mx, p.my, p.radius, tiles_x, tiles_y, e);
            ++kept;
            pairs += rect_count(e);
            for (int ty = e.ty0; ty <= e.ty1; ++ty)
                for (int tx = e.tx0; tx <= e.tx1; ++tx) {
                    const unsigned tile = unsigned(ty * tiles_x + tx);
                    const unsigned long long key =
                        (unsigned long long)tile << 32 | e.depth_bits;
                    kor |= key;
                    knand |= ~key;
                    if (use_hist)
                        atomicAdd(s_hist + tile, 1u);
                    else
                        atomicAdd(out.tile_count + tile, 1u);
                }
        } else {
            e.depth_bits = 0;
            e.tx0 = 1;
            e.tx1 = 0;
            e.ty0 = kDropped;
            e.ty1 = 0;
        }
        out.emit[s] = e;
    }
    block_add2(kept, pairs, &cnt->n_gaussians, &cnt->n_pairs);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        kor |= __shfl_xor_sync(0xffffffffu, kor, off);
        knand |= __shfl_xor_sync(0xffffffffu, knand, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (kor) atomicOr(&cnt->key_or, kor);
        if (knand) atomicOr(&cnt->key_nand, knand);
    }
    if (use_hist) {
        __shared__ uint32_t s_nlist;
        if (threadIdx.x == 0) s_nlist = 0u;
        __syncthreads();
        uint2* list = out.tile_lists ? out.tile_lists + uint64_t(blockIdx.x) * n_tiles : nullptr;
        const unsigned lane = threadIdx.x & 31;
        for (int t0 = 0; t0 < n_tiles; t0 += kPrepBlock) {  // warp-uniform trip count
            const int t = t0 + int(threadIdx.x);
            const uint32_t c = t < n_tiles ? s_hist[t] : 0u;
            if (c) atomicAdd(out.tile_count + t, c);
            if (list) {  // compacted append, one shared atomic per warp
                const unsigned m = __ballot_sync(0xffffffffu, c != 0u);
                uint32_t base = 0;
                if (lane == 0 && m) base = atomicAdd(&s_nlist, unsigned(__popc(m)));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (c) list[base + __popc(m & ((1u << lane) - 1u))] = make_uint2(uint32_t(t), c);
            }
        }
        if (list) {
            __syncthreads();
            if (threadIdx.x == 0) out.tile_list_len[blockIdx.x] = s_nlist;
        }
    }
}

// ---------------------------------------------------------------------------
// View-dependent colour (SH degree 1..3, lodgs_gpu_scene_set_sh): an extension for
// BASELINE configs[1] ("SH deg 3").  The reference is SH0-only (SPEC.md:78,
// scene.hpp:15-24), so there is no reference colour to match; the evaluation is
// the standard real SH basis of 3D Gaussian splatting (constants below) on top of the
// node's SH0 colour, clamped at 0:
//     colour = max(rgb + sum_k c_k Y_k(d), 0),  d = (mean - camera centre) * (1 / |.|)
// in FP64, every operation in the order written (-fmad=false), so
// tests/test_gpu_sh.py restates it in numpy bit for bit.  With all c_k = 0 the sum
// adds +-0 and, for rgb >= 0, the colour is rgb exactly: the SH0 frame.  Runs
// after K3 over the frame's slots and rewrites the colours of the kept ones
// (Gauss32 r/g/b, and the FP64 colours of the exact blend when present).
__constant__ double kShC1 = 0.4886025119029199;
__constant__ double kShC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                               -1.0925484305920792, 0.5462742152960396};
__constant__ double kShC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                               0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                               -0.5900435899266435};

// Y_k(d) for the K = 3 / 8 / 15 rest coefficients, each product left to right.
template <int K>
__device__ __forceinline__ void sh_basis(double x, double y, double z, double (&Y)[K]) {
    Y[0] = -kShC1 * y;
    Y[1] = kShC1 * z;
    Y[2] = -kShC1 * x;
    if constexpr (K > 3) {
        const double xx = x * x, yy = y * y, zz = z * z;
        Y[3] = kShC2[0] * (x * y);
        Y[4] = kShC2[1] * (y * z);
        Y[5] = kShC2[2] * (2.0 * zz - xx - yy);
        Y[6] = kShC2[3] * (x * z);
        Y[7] = kShC2[4] * (xx - yy);
        if constexpr (K > 8) {
            Y[8] = kShC3[0] * y * (3.0 * xx - yy);
            Y[9] = kShC3[1] * (x * y) * z;
            Y[10] = kShC3[2] * y * (4.0 * zz - xx - yy);
            Y[11] = kShC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            Y[12] = kShC3[4] * x * (4.0 * zz - xx - yy);
            Y[13] = kShC3[5] * z * (xx - yy);
            Y[14] = kShC3[6] * x * (xx - 3.0 * yy);
        }
    }
}

#ifndef SH_MIN_CTAS
#define SH_MIN_CTAS 1
#endif
template <int K>
__global__ void __launch_bounds__(kPrepBlock, SH_MIN_CTAS) k_sh_colour(
    const Geom g, const SplatRec* __restrict__ splat, const float4* __restrict__ sh,
    const GaussEmit* __restrict__ emit, Gauss32* g32, GaussCol64* col64,
    const FrameCounters* __restrict__ cnt) {
    pdl_wait();  // K3 is complete and visible
    pdl_trigger();
    constexpr int kStride = (3 * K + 3) / 4;  // float4s per node
    // camera centre in world space: -R^T t (CameraGeom's world-to-camera R, t)
    const double cx = -((g.rot[0] * g.trans[0] + g.rot[3] * g.trans[1]) + g.rot[6] * g.trans[2]);
    const double cy = -((g.rot[1] * g.trans[0] + g.rot[4] * g.trans[1]) + g.rot[7] * g.trans[2]);
    const double cz = -((g.rot[2] * g.trans[0] + g.rot[5] * g.trans[1]) + g.rot[8] * g.trans[2]);
    const uint64_t n = cnt->n_selected;
    for (uint64_t s = uint64_t(blockIdx.x) * kPrepBlock + threadIdx.x; s < n;
         s += uint64_t(gridDim.x) * kPrepBlock) {
        const GaussEmit e = emit[s];
        if (e.ty0 == kDropped) continue;
        const float4* rec = reinterpret_cast<const float4*>(splat + e.node);
        const float4 m = __ldg(rec), c3 = __ldg(rec + 2), c4 = __ldg(rec + 3);  // mean; cr; cg, cb
        float c[4 * kStride];
        const float4* row = sh + uint64_t(e.node) * kStride;
#pragma unroll
        for (int j = 0; j < kStride; ++j) {
            const float4 v = __ldg(row + j);
            c[4 * j] = v.x;
            c[4 * j + 1] = v.y;
            c[4 * j + 2] = v.z;
            c[4 * j + 3] = v.w;
        }
        const double dx = double(m.x) - cx, dy = double(m.y) - cy, dz = double(m.z) - cz;
        const double inv = 1.0 / sqrt((dx * dx + dy * dy) + dz * dz);
        double Y[K];
        sh_basis<K>(dx * inv, dy * inv, dz * inv, Y);
        double r = double(c3.w), gg = double(c4.x), b = double(c4.y);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            r = r + Y[k] * double(c[3 * k]);
            gg = gg + Y[k] * double(c[3 * k + 1]);
            b = b + Y[k] * double(c[3 * k + 2]);
        }
        r = r < 0.0 ? 0.0 : r;
        gg = gg < 0.0 ? 0.0 : gg;
        b = b < 0.0 ? 0.0 : b;
        g32[s].r = float(r);
        g32[s].g = float(gg);
        g32[s].b = float(b);
        if (col64) {
            col64[s].r = r;
            col64[s].g = gg;
            col64[s].b = b;
        }
    }
}

void launch_sh_colour(const Geom& g, const DevTree& t, const GaussEmit* emit, Gauss32* g32,
                      GaussCol64* col64, const FrameCounters* cnt, int grid, cudaStream_t s) {
    if (!t.sh || t.sh_k <= 0) return;
    if (t.sh_k == 3)
        launch_pdl(k_sh_colour<3>, grid, kPrepBlock, 0, s, g, t.splat, t.sh, emit, g32, col64, cnt);
    else if (t.sh_k == 8)
        launch_pdl(k_sh_colour<8>, grid, kPrepBlock, 0, s, g, t.splat, t.sh, emit, g32, col64, cnt);
    else
        launch_pdl(k_sh_colour<15>, grid, kPrepBlock, 0, s, g, t.splat, t.sh, emit, g32, col64, cnt);
}

void launch_preprocess(const Geom& g, const DevTree& t, const uint32_t* selected,
                       uint64_t max_selected, int shrink_kind, double tau, int tiles_x,
                       int tiles_y, PrepOut out, FrameCounters* cnt, int grid, cudaStream_t s,
                       bool known_visible) {
    if (max_selected == 0) return;
    const int n_tiles = tiles_x * tiles_y;
    const int use_hist = n_tiles <= kHistMaxTiles ? 1 : 0;
    const size_t smem = use_hist ? size_t(n_tiles) * 4 : 0;
    // the tile histogram plus the kernel's static shared memory can pass the
    // default 48 KB per-block limit near kHistMaxTiles (a 2048x1536 frame)
    opt_in_smem(k_preprocess, kHistMaxTiles * 4 + 1024);
    launch_pdl(k_preprocess, grid, kPrepBlock, smem, s, g, t.splat,
               selected, shrink_kind, tau, tiles_x, tiles_y,
               out, cnt, use_hist, known_visible ? 1 : 0);
}

// One CTA: exclusive scan of per-tile counts -> offsets and write cursors,
// the list of tiles too large for the shared-memory sort, the heavy-first
// schedule for the per-tile grids, and (optionally) the running totals.
// Thread k owns the contiguous tiles [k*per, (k+1)*per): a serial sum, one
// block scan, a serial write-back.
// SURVEY.md 8(d) sort bytes of the reference's LSD radix (rasterizer.cpp:
// 100-135): 24 B per pair for every 8-bit digit that is not uniform across
// the frame's keys (uniform digits are skipped, :117), plus 8 B per pair for
// the histogram pass.
__device__ __forceinline__ unsigned long long sort_bytes(const FrameCounters* cnt,
                                                         unsigned long long n_pairs) {
    const unsigned long long diff = cnt->key_or & cnt->key_nand;  // bits that differ
    int passes = 0;
#pragma unroll
    for (int d = 0; d < 8; ++d) passes += ((diff >> (8 * d)) & 0xffull) ? 1 : 0;
    return (24ull * unsigned(passes) + 8ull) * n_pairs;
}

// Running totals with fire-and-forget reductions: the counters are read once (one
// round trip, the loads independent) and nothing waits on the RMWs.
__device__ __forceinline__ void add_totals(RunTotals* totals, const FrameCounters* cnt,
                                           unsigned long long total, bool ovf) {
    const unsigned long long sel = cnt->n_selected;
    const unsigned long long sb = ovf ? 0ull : sort_bytes(cnt, total);
    atomicAdd(&totals->frames, 1ull);
    atomicAdd(&totals->sum_selected, sel);
    if (!ovf) atomicAdd(&totals->sum_pairs, total);
    if (ovf) atomicOr(&totals->pad, 1ull);
    if (sb) atomicAdd(&totals->sum_sort_bytes, sb);
}

// The frame's final counters into the batch log, one 8-byte word per thread.
__device__ __forceinline__ void copy_counters(FrameCounters* log, const FrameCounters* cnt,
                                              unsigned tid) {
    constexpr unsigned kWords = sizeof(FrameCounters) / 8;
    static_assert(sizeof(FrameCounters) % 8 == 0, "FrameCounters is a whole number of words");
    if (tid < kWords)
        reinterpret_cast<unsigned long long*>(log)[tid] =
            reinterpret_cast<const volatile unsigned long long*>(cnt)[tid];
}

__device__ __forceinline__ int tile_class(uint32_t c, uint32_t mean) {
    // 0: >= 4x mean pairs, 1: >= 2x, 2: >= 1x, 3: lighter
    return c >= 4 * mean ? 0 : (c >= 2 * mean ? 1 : (c >= mean ? 2 : 3));
}

__global__ void __launch_bounds__(1024) k_tile_offsets(const uint32_t* __restrict__ gcount,
                                                       int n_tiles, uint32_t* offsets,
                                                       uint32_t* cursor, uint32_t* big_list,
                                                       uint32_t* order, FrameCounters* cnt,
                                                       uint64_t pair_cap, RunTotals* totals,
                                                       int staged, FrameCounters* log) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    // staged: counts, then offsets, in s_buf[0, n]; the order in s_buf[n+1, 2n+1).
    // Every global write then leaves the SM as coalesced rows -- a single SM's
    // scattered stores were the bottleneck of this kernel (~1 sector/clk).
    __shared__ uint64_t s_warp[32];
    __shared__ uint32_t s_cls[4][32];  // per (class, warp): tiles, then first order slot
    extern __shared__ uint32_t s_buf[];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* off = staged ? s_buf : offsets;
    uint32_t* ord = staged ? s_buf + n_tiles + 1 : order;
    if (staged) {
#pragma unroll 8
        for (int t = threadIdx.x; t < n_tiles; t += 1024) s_buf[t] = __ldg(gcount + t);
        __syncthreads();
    }
    const uint32_t* count = staged ? s_buf : gcount;
    const int per = (n_tiles + 1023) / 1024;
    const int t0 = min(n_tiles, int(threadIdx.x) * per), t1 = min(n_tiles, t0 + per);
    uint64_t sum = 0;
    for (int t = t0; t < t1; ++t) sum += count[t];
    uint64_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= unsigned(o)) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint64_t v = s_warp[lane];
        uint64_t wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t u = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= unsigned(o)) wi += u;
        }
        s_warp[lane] = wi;  // inclusive warp prefix
    }
    __syncthreads();
    const uint64_t total = s_warp[31];
    // Overflow: every bucket becomes empty so sort/blend never touch the
    // unwritten keys; the host grows the buffer and re-renders.
    const bool ovf = total > pair_cap;
    uint64_t run = (warp ? s_warp[warp - 1] : 0ull) + (incl - sum);
    for (int t = t0; t < t1; ++t) {
        const uint32_t c = count[t];  // staged: read before the in-place overwrite
        off[t] = ovf ? 0u : uint32_t(run);
        run += c;
        if (!ovf && c > uint32_t(kSmallSortCap))
            big_list[atomicAdd(&cnt->big_tiles, 1u)] = uint32_t(t);
    }
    if (threadIdx.x == 0) {
        off[n_tiles] = ovf ? 0u : uint32_t(total);
        if (ovf) cnt->overflow = 1u;
        if (totals) add_totals(totals, cnt, total, ovf);
    }
    __syncthreads();
    if (staged) {
        for (int t = threadIdx.x; t <= n_tiles; t += 1024) {
            const uint32_t o = s_buf[t];
            offsets[t] = o;
            if (t < n_tiles) cursor[t] = o;
        }
    } else {
        for (int t = threadIdx.x; t < n_tiles; t += 1024) cursor[t] = offsets[t];
    }
    // Heavy-first schedule for the per-tile kernels (sort, blend): a stable
    // partition of the tiles into four classes by pair count relative to the
    // mean, heaviest class first, so the longest CTAs start first and the
    // tail of the grid is made of cheap ones.  Warp ballots count and rank
    // (no atomics).  The order only schedules work; it never changes a result.
    const uint32_t mean = uint32_t(total / uint64_t(n_tiles > 0 ? n_tiles : 1)) + 1u;
    const int rounds = (n_tiles + 1023) / 1024;
    unsigned my_cnt = 0;  // lane c < 4: tiles of class c seen by this warp
    for (int k = 0; k < rounds; ++k) {
        const int t = k * 1024 + int(threadIdx.x);
        const int cls = t < n_tiles ? tile_class(off[t + 1] - off[t], mean) : 4;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned m = __ballot_sync(0xffffffffu, cls == c);
            if (lane == unsigned(c)) my_cnt += __popc(m);
        }
    }
    if (lane < 4) s_cls[lane][warp] = my_cnt;
    __syncthreads();
    if (warp < 4) {  // warp c scans class c over the 32 warps
        const uint32_t v = s_cls[warp][lane];
        uint32_t wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= unsigned(o)) wi += u;
        }
        s_cls[warp][lane] = wi - v;
        if (lane == 31) s_warp[warp] = wi;  // class total (s_warp is free again)
    }
    __syncthreads();
    uint32_t rank[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t before = 0;
        for (int d = 0; d < c; ++d) before += uint32_t(s_warp[d]);
        rank[c] = before + s_cls[c][warp];
    }
    const unsigned lt = (1u << lane) - 1u;
    for (int k = 0; k < rounds; ++k) {
        const int t = k * 1024 + int(threadIdx.x);
        const int cls = t < n_tiles ? tile_class(off[t + 1] - off[t], mean) : 4;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned m = __ballot_sync(0xffffffffu, cls == c);
            if (cls == c) ord[rank[c] + __popc(m & lt)] = uint32_t(t);
            rank[c] += __popc(m);
        }
    }
    if (staged) {
        __syncthreads();
        for (int t = threadIdx.x; t < n_tiles; t += 1024) order[t] = ord[t];
    }
    __syncthreads();
    if (log) copy_counters(log, cnt, threadIdx.x);
}

// Cluster variant for up to 8 x 12,288 tiles: the 8 CTAs of one thread-block
// cluster each own a contiguous chunk of tiles, and exchange their chunk
// totals and class counts through distributed shared memory (two cluster
// barriers) -- the single-CTA kernel above is bound by one SM's issue rate.
namespace cg = cooperative_groups;
constexpr int kOffCtas = 8;
constexpr int kOffChunkMax = 12288;

__global__ void __cluster_dims__(kOffCtas, 1, 1) __launch_bounds__(1024) k_tile_offsets_cluster(
    const uint32_t* __restrict__ gcount, int n_tiles, uint32_t* offsets, uint32_t* cursor,
    uint32_t* big_list, uint32_t* order, FrameCounters* cnt, uint64_t pair_cap,
    RunTotals* totals, FrameCounters* log) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned crank = cluster.block_rank();
    __shared__ unsigned long long s_tot;  // this chunk's pair total (read by every CTA)
    __shared__ uint32_t s_ccls[4];        // this chunk's tiles per class (read by every CTA)
    __shared__ uint64_t s_warp[32];
    __shared__ uint32_t s_wcls[4][32];
    extern __shared__ uint32_t s_off[];  // chunk counts, then offsets; [m] = chunk end
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int chunk = (n_tiles + kOffCtas - 1) / kOffCtas;
    const int c0 = min(n_tiles, int(crank) * chunk), m = min(n_tiles, c0 + chunk) - c0;
#pragma unroll 4
    for (int t = threadIdx.x; t < m; t += 1024) s_off[t] = __ldg(gcount + c0 + t);
    __syncthreads();
    const int per = (chunk + 1023) / 1024;
    const int t0 = min(m, int(threadIdx.x) * per), t1 = min(m, t0 + per);
    uint64_t sum = 0;
    for (int t = t0; t < t1; ++t) sum += s_off[t];
    uint64_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= unsigned(o)) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint64_t v = s_warp[lane];
        uint64_t wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t u = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= unsigned(o)) wi += u;
        }
        s_warp[lane] = wi;
        if (lane == 31) s_tot = wi;
    }
    cluster.sync();  // #1: chunk totals visible cluster-wide
    uint64_t total = 0, base = 0;
#pragma unroll
    for (int r = 0; r < kOffCtas; ++r) {
        const uint64_t v = *cluster.map_shared_rank(&s_tot, r);
        total += v;
        base += unsigned(r) < crank ? v : 0ull;
    }
    // Overflow: every bucket becomes empty so sort/blend never touch the
    // unwritten keys; the host grows the buffer and re-renders.
    const bool ovf = total > pair_cap;
    uint64_t run = base + (warp ? s_warp[warp - 1] : 0ull) + (incl - sum);
    for (int t = t0; t < t1; ++t) {
        const uint32_t c = s_off[t];
        s_off[t] = ovf ? 0u : uint32_t(run);
        run += c;
        if (!ovf && c > uint32_t(kSmallSortCap))
            big_list[atomicAdd(&cnt->big_tiles, 1u)] = uint32_t(c0 + t);
    }
    if (threadIdx.x == 0) s_off[m] = ovf ? 0u : uint32_t(base + s_tot);
    __syncthreads();
    for (int t = threadIdx.x; t < m; t += 1024) {
        const uint32_t o = s_off[t];
        offsets[c0 + t] = o;
        cursor[c0 + t] = o;
    }
    if (threadIdx.x == 0 && c0 + m == n_tiles && m > 0) offsets[n_tiles] = s_off[m];
    if (crank == 0 && threadIdx.x == 0) {
        if (n_tiles == 0) offsets[0] = 0u;
        if (ovf) cnt->overflow = 1u;
        if (totals) add_totals(totals, cnt, total, ovf);
    }
    // heavy-first schedule (see k_tile_offsets): classes by count vs the mean
    const uint32_t mean = uint32_t(total / uint64_t(n_tiles > 0 ? n_tiles : 1)) + 1u;
    unsigned my_cnt = 0;
    for (int k = 0; k < per; ++k) {
        const int t = k * 1024 + int(threadIdx.x);
        const int cls = t < m ? tile_class(s_off[t + 1] - s_off[t], mean) : 4;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned msk = __ballot_sync(0xffffffffu, cls == c);
            if (lane == unsigned(c)) my_cnt += __popc(msk);
        }
    }
    if (lane < 4) s_wcls[lane][warp] = my_cnt;
    __syncthreads();
    if (warp < 4) {  // warp c scans class c over the 32 warps
        const uint32_t v = s_wcls[warp][lane];
        uint32_t wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= unsigned(o)) wi += u;
        }
        s_wcls[warp][lane] = wi - v;
        if (lane == 31) s_ccls[warp] = wi;
    }
    cluster.sync();  // #2: chunk class counts visible cluster-wide
    uint32_t rank[4];
    {
        uint32_t all[4] = {0u, 0u, 0u, 0u}, before[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int r = 0; r < kOffCtas; ++r) {
            const uint32_t* rc = cluster.map_shared_rank(s_ccls, r);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t v = rc[c];
                all[c] += v;
                before[c] += unsigned(r) < crank ? v : 0u;
            }
        }
        uint32_t cb = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            rank[c] = cb + before[c] + s_wcls[c][warp];
            cb += all[c];
        }
    }
    const unsigned lt = (1u << lane) - 1u;
    for (int k = 0; k < per; ++k) {
        const int t = k * 1024 + int(threadIdx.x);
        const int cls = t < m ? tile_class(s_off[t + 1] - s_off[t], mean) : 4;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned msk = __ballot_sync(0xffffffffu, cls == c);
            if (cls == c) order[rank[c] + __popc(msk & lt)] = uint32_t(c0 + t);
            rank[c] += __popc(msk);
        }
    }
    cluster.sync();  // no CTA leaves while its shared memory may still be read
    // the frame's final counters into the batch log (no per-frame D2H on the
    // compute stream: a D2H there would queue behind the image copies)
    if (log && crank == 0) copy_counters(log, cnt, threadIdx.x);
}

void launch_tile_offsets(const uint32_t* tile_count, int n_tiles, uint32_t* offsets,
                         uint32_t* cursor, uint32_t* big_list, uint32_t* order,
                         FrameCounters* cnt, uint64_t pair_cap, cudaStream_t s,
                         RunTotals* totals, FrameCounters* log) {
    if (n_tiles <= kOffCtas * kOffChunkMax) {
        const int chunk = (n_tiles + kOffCtas - 1) / kOffCtas;
        const size_t smem = size_t(chunk + 1) * 4;
        if (smem > 48 * 1024) {
            static bool attr_set[64] = {};  // function attributes are per device
            int dev = 0;
            cudaGetDevice(&dev);
            if (dev < 0 || dev >= 64 || !attr_set[dev]) {
                cudaFuncSetAttribute(k_tile_offsets_cluster,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (kOffChunkMax + 1) * 4);
                if (dev >= 0 && dev < 64) attr_set[dev] = true;
            }
        }
        launch_pdl(k_tile_offsets_cluster, kOffCtas, 1024, smem, s, tile_count, n_tiles, offsets,
                   cursor, big_list, order, cnt, pair_cap, totals, log);
        return;
    }
    // beyond 98,304 tiles (> 8K frames): one CTA, global memory
    const int staged = 0;
    const size_t smem = 0;
    k_tile_offsets<<<1, 1024, smem, s>>>(tile_count, n_tiles, offsets, cursor, big_list, order,
                                         cnt, pair_cap, totals, staged, log);
}

// Key duplication with CTA-level aggregation: each CTA counts its slice's
// pairs per tile in shared memory, reserves one contiguous run per touched
// tile with a single global atomic, then scatters its keys into the runs.
__global__ void __launch_bounds__(256) k_emit_keys(const GaussEmit* __restrict__ emit,
                                                   const FrameCounters* cnt, int tiles_x,
                                                   int n_tiles, uint32_t* cursor,
                                                   unsigned long long* keys, int use_hist,
                                                   const uint2* __restrict__ tile_lists,
                                                   const uint32_t* __restrict__ tile_list_len) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    extern __shared__ uint32_t s_hist[];
    if (cnt->overflow) return;
    uint64_t lo, hi;
    cta_range(cnt->n_selected, lo, hi);
    if (!use_hist) {
        for (uint64_t s = lo + threadIdx.x; s < hi; s += blockDim.x) {
            const GaussEmit e = emit[s];
            const unsigned long long key = (unsigned long long)e.depth_bits << 32 | s;
            for (int ty = e.ty0; ty <= e.ty1; ++ty)
                for (int tx = e.tx0; tx <= e.tx1; ++tx)
                    keys[atomicAdd(cursor + (ty * tiles_x + tx), 1u)] = key;
        }
        return;
    }
    if (tile_lists) {
        // K3 left this CTA's nonzero (tile, count) entries (same slice, same grid):
        // reserve one run per touched tile; untouched tiles are never read below
        const uint2* list = tile_lists + uint64_t(blockIdx.x) * n_tiles;
        const uint32_t nl = tile_list_len[blockIdx.x];
        for (uint32_t k = threadIdx.x; k < nl; k += blockDim.x) {
            const uint2 e = list[k];
            s_hist[e.x] = atomicAdd(cursor + e.x, e.y);
        }
    } else {
        for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) s_hist[t] = 0u;
        __syncthreads();
        for (uint64_t s = lo + threadIdx.x; s < hi; s += blockDim.x) {
            const GaussEmit e = emit[s];
            for (int ty = e.ty0; ty <= e.ty1; ++ty)
                for (int tx = e.tx0; tx <= e.tx1; ++tx)
                    atomicAdd(s_hist + (ty * tiles_x + tx), 1u);
        }
        __syncthreads();
        for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
            const uint32_t c = s_hist[t];
            if (c) s_hist[t] = atomicAdd(cursor + t, c);
        }
    }
    __syncthreads();
    for (uint64_t s = lo + threadIdx.x; s < hi; s += blockDim.x) {
        const GaussEmit e = emit[s];
        const unsigned long long key = (unsigned long long)e.depth_bits << 32 | s;
        for (int ty = e.ty0; ty <= e.ty1; ++ty)
            for (int tx = e.tx0; tx <= e.tx1; ++tx)
                keys[atomicAdd(s_hist + (ty * tiles_x + tx), 1u)] = key;
    }
}

void launch_emit_keys(const GaussEmit* emit, const FrameCounters* cnt, int tiles_x, int n_tiles,
                      uint32_t* cursor, unsigned long long* keys, int grid, cudaStream_t s,
                      const uint2* tile_lists, const uint32_t* tile_list_len) {
    const int use_hist = n_tiles <= kHistMaxTiles ? 1 : 0;
    const size_t smem = use_hist ? size_t(n_tiles) * 4 : 0;
    opt_in_smem(k_emit_keys, kHistMaxTiles * 4 + 1024);
    launch_pdl(k_emit_keys, grid, 256, smem, s, emit, cnt, tiles_x, n_tiles, cursor, keys,
               use_hist, use_hist ? tile_lists : nullptr, use_hist ? tile_list_len : nullptr);
}

// Readback support: slot -> BlendList index (chained scan over kept flags),
// and the inverse list.
__global__ void __launch_bounds__(256) k_slot_map(const GaussEmit* __restrict__ emit,
                                                  uint64_t n, unsigned long long* status,
                                                  FrameCounters* cnt, uint32_t* g_of_slot,
                                                  uint32_t* slot_of_g) {
    __shared__ unsigned s_ticket;
    __shared__ unsigned s_warp[8];
    __shared__ unsigned long long s_excl;
    const unsigned n_tiles = unsigned((n + 255) / 256);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    while (true) {
        const unsigned tile = take_ticket(&cnt->ticket_prep, &s_ticket);
        if (tile >= n_tiles) break;
        const uint64_t s = uint64_t(tile) * 256 + threadIdx.x;
        const bool kept = s < n && emit[s].ty0 != kDropped;
        const unsigned km = __ballot_sync(0xffffffffu, kept);
        if (lane == 0) s_warp[warp] = __popc(km);
        __syncthreads();
        if (warp == 0) {
            unsigned v = lane < 8 ? s_warp[lane] : 0u;
            unsigned incl = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const unsigned o = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= unsigned(off)) incl += o;
            }
            const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
            if (lane < 8) s_warp[lane] = incl - v;
            const unsigned long long excl = chained_scan_warp(status, tile, total);
            if (lane == 0) s_excl = excl;
        }
        __syncthreads();
        if (s < n) {
            if (kept) {
                const uint32_t gi = uint32_t(s_excl + s_warp[warp] + __popc(km & ((1u << lane) - 1u)));
                g_of_slot[s] = gi;
                slot_of_g[gi] = uint32_t(s);
            } else {
                g_of_slot[s] = 0xFFFFFFFFu;
            }
        }
    }
}

void launch_slot_map(const GaussEmit* emit, uint64_t n, unsigned long long* status,
                     FrameCounters* cnt, uint32_t* g_of_slot, uint32_t* slot_of_g, int grid,
                     cudaStream_t s) {
    if (n) k_slot_map<<<grid, 256, 0, s>>>(emit, n, status, cnt, g_of_slot, slot_of_g);
}

__global__ void k_compact_records(const uint32_t* slot_of_g, uint64_t n_g, const Gauss64* g64,
                                  const Gauss32* g32, const GaussEmit* emit, Gauss64* o64,
                                  Gauss32* o32, GaussEmit* oe) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_g) return;
    const uint32_t s = slot_of_g[i];
    o64[i] = g64[s];
    o32[i] = g32[s];
    oe[i] = emit[s];
}

void launch_compact_records(const uint32_t* slot_of_g, uint64_t n_g, const Gauss64* g64,
                            const Gauss32* g32, const GaussEmit* emit, Gauss64* o64, Gauss32* o32,
                            GaussEmit* oe, cudaStream_t s) {
    if (n_g)
        k_compact_records<<<unsigned((n_g + 255) / 256), 256, 0, s>>>(slot_of_g, n_g, g64, g32,
                                                                    emit, o64, o32, oe);
}

// ----------------------------------------------------------------------------
// Stage-entry helpers.

// bin_to_tiles in the reference's emission order (rasterizer.cpp:75-98):
// gaussian-major, row-major tiles.  Chained scan of per-gaussian counts.
__global__ void __launch_bounds__(256) k_bin_reference_order(
    const GaussEmit* __restrict__ emit, uint64_t n, int tiles_x, unsigned long long* status,
    FrameCounters* cnt, uint32_t* out, uint64_t cap) {
    __shared__ unsigned s_ticket;
    __shared__ unsigned long long s_warp[8];
    __shared__ unsigned long long s_excl;
    const unsigned n_scan_tiles = unsigned((n + 255) / 256);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    while (true) {
        const unsigned tile = take_ticket(&cnt->ticket_bin, &s_ticket);
        if (tile >= n_scan_tiles) break;
        const uint64_t gi = uint64_t(tile) * 256 + threadIdx.x;
        GaussEmit e;
        e.tx0 = 0; e.tx1 = -1; e.ty0 = 0; e.ty1 = -1; e.depth_bits = 0;
        if (gi < n) e = emit[gi];
        const unsigned long long c = rect_count(e);
        unsigned long long incl = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned long long o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= unsigned(off)) incl += o;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            unsigned long long v = lane < 8 ? s_warp[lane] : 0ull;
            unsigned long long wi = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const unsigned long long o = __shfl_up_sync(0xffffffffu, wi, off);
                if (lane >= unsigned(off)) wi += o;
            }
            const unsigned long long total = __shfl_sync(0xffffffffu, wi, 31);
            if (lane < 8) s_warp[lane] = wi - v;
            const unsigned long long excl = chained_scan_warp(status, tile, total);
            if (lane == 0) {
                s_excl = excl;
                if (tile == n_scan_tiles - 1) cnt->n_pairs = excl + total;
            }
        }
        __syncthreads();
        if (out) {
            uint64_t pos = s_excl + s_warp[warp] + (incl - c);
            for (int ty = e.ty0; ty <= e.ty1; ++ty)
                for (int tx = e.tx0; tx <= e.tx1; ++tx, ++pos)
                    if (pos < cap) {
                        out[pos * 3 + 0] = uint32_t(ty) * uint32_t(tiles_x) + uint32_t(tx);
                        out[pos * 3 + 1] = e.depth_bits;
                        out[pos * 3 + 2] = uint32_t(gi);
                    }
        }
    }
}

void launch_bin_reference_order(const GaussEmit* emit, uint64_t n, int tiles_x,
                                unsigned long long* status, FrameCounters* cnt,
                                uint32_t* out_triples, uint64_t cap, int grid, cudaStream_t s) {
    if (n == 0) return;
    k_bin_reference_order<<<grid, 256, 0, s>>>(emit, n, tiles_x, status, cnt, out_triples, cap);
}

__global__ void k_pack_blendlist(uint64_t n, const double* mx, const double* my, const double* ca,
                                 const double* cb, const double* cc, const double* op,
                                 const double* cr, const double* cg, const double* cbl,
                                 const double* radius, const float* depth, int tiles_x,
                                 int tiles_y, Gauss64* g64, Gauss32* g32, GaussCol64* col64,
                                 GaussEmit* emit) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Gauss64 r;
    r.ca = ca[i];
    r.cb = cb[i];
    r.cc = cc[i];
    r.op = op[i];
    g64[i] = r;
    const double rad = radius ? radius[i] : 0.0;
    if (col64) {
        GaussCol64 c;
        c.r = cr[i];
        c.g = cg[i];
        c.b = cbl[i];
        c.pad = 0.0;
        col64[i] = c;
    }
    g32[i] = make_g32(ca[i], cb[i], cc[i], op[i], cr[i], cg[i], cbl[i], mx[i], my[i], rad);
    if (emit) {
        GaussEmit e;
        e.depth_bits = __float_as_uint(depth[i]);
        e.node = uint32_t(i);
        tile_rect(mx[i], my[i], rad, tiles_x, tiles_y, e);
        emit[i] = e;
    }
}

void launch_pack_blendlist(uint64_t n, const double* mx, const double* my, const double* ca,
                           const double* cb, const double* cc, const double* op,
                           const double* cr, const double* cg, const double* cbl,
                           const double* radius, const float* depth, int tiles_x, int tiles_y,
                           Gauss64* g64, Gauss32* g32, GaussCol64* col64, GaussEmit* emit,
                           cudaStream_t s) {
    if (n == 0) return;
    k_pack_blendlist<<<unsigned((n + 255) / 256), 256, 0, s>>>(
        n, mx, my, ca, cb, cc, op, cr, cg, cbl, radius, depth, tiles_x, tiles_y, g64, g32, col64,
        emit);
}

__global__ void k_gauss_counts(const GaussEmit* emit, const FrameCounters* cnt, uint64_t cap,
                               uint32_t* out) {
    const uint64_t n = cnt->n_gaussians < cap ? cnt->n_gaussians : cap;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = rect_count(emit[i]);
}

void launch_gauss_counts(const GaussEmit* emit, const FrameCounters* cnt, uint64_t cap,
                         uint32_t* out, cudaStream_t s) {
    k_gauss_counts<<<296, 256, 0, s>>>(emit, cnt, cap, out);
}

}  // namespace fgs
