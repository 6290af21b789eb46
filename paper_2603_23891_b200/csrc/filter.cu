// filter.cu -- the traversal-free parallel LoD filter (FilterGS),
// reference filter_parallel (filter.cpp:115-150).
//
// K1 mark: one flat coalesced pass over the SoA arena.  Per node: camera
// transform + sphere-vs-frustum (FP64, exact), and -- only for visible,
// projectable internal nodes -- the EWA radius.  A leaf's qpass is never
// read by the selection rule (candidates use vis && (qpass || leaf),
// ancestors use qpass && !leaf, filter.cpp:23,137), so leaves and culled
// nodes skip the covariance entirely.  Output: two bitmasks written by warp
// ballot, cand = vis && (qpass || leaf) and qint = qpass && !leaf.
//
// K2 select: candidates walk their parent chain against the L2-resident qint
// bitmask (filter.cpp:20-25); survivors are compacted in node order by a
// single-pass chained scan, so `selected` comes out strictly increasing as
// filter.cpp:147-148 produces it.
#include "launch.h"
#include "mark.cuh"
#include "scan.cuh"

namespace fgs {

// FP32 copy of the camera for the certified pre-test.
struct GeomF {
    float r[9], t[3];
    float p2x, p2z, p3x, p3z, p4y, p4z, p5y, p5z;  // side-plane coefficients
    float znear, zfar;
    float c0;  // max(|t_i|, znear, zfar) + 1: magnitude term of the error bound
};

GeomF make_geomf(const Geom& g) {
    GeomF f;
    for (int i = 0; i < 9; ++i) f.r[i] = float(g.rot[i]);
    double c0 = 0.0;
    for (int i = 0; i < 3; ++i) {
        f.t[i] = float(g.trans[i]);
        c0 = fmax(c0, fabs(g.trans[i]));
    }
    f.p2x = float(g.planes[2][0]);
    f.p2z = float(g.planes[2][2]);
    f.p3x = float(g.planes[3][0]);
    f.p3z = float(g.planes[3][2]);
    f.p4y = float(g.planes[4][1]);
    f.p4z = float(g.planes[4][2]);
    f.p5y = float(g.planes[5][1]);
    f.p5z = float(g.planes[5][2]);
    f.znear = float(g.znear);
    f.zfar = float(g.zfar);
    f.c0 = float(fmax(c0, fmax(g.znear, g.zfar)) + 1.0);
    return f;
}

// Certified FP32 frustum pre-test.  With |R_ij| <= 1 and unit plane normals,
// every FP32 camera-space coordinate is within B = 2^-20 (|x|+|y|+|z|+c0) of
// the exact value (16 ulp of the magnitude sum, covering coefficient
// rounding and the three FMA roundings), and every plane distance within
// 3B + 2^-22 |.|.  When min_p(d_p + r3) clears +-E, E = 4B + 2^-22 r3, the
// FP64 reference decision (mark_core.hpp:32-40) is certain; only the
// remainder (nodes within ~1e-3 world units of a frustum plane) recompute in
// FP64.  Returns 1 visible, 0 culled, -1 undecided; *zs likewise for z_ok.
__device__ __forceinline__ int frustum_fp32(const GeomF& f, float mx, float my, float mz,
                                            float r3, float& tz_out, int& zs) {
    const float tx = __fmaf_rn(f.r[0], mx, __fmaf_rn(f.r[1], my, __fmaf_rn(f.r[2], mz, f.t[0])));
    const float ty = __fmaf_rn(f.r[3], mx, __fmaf_rn(f.r[4], my, __fmaf_rn(f.r[5], mz, f.t[1])));
    const float tz = __fmaf_rn(f.r[6], mx, __fmaf_rn(f.r[7], my, __fmaf_rn(f.r[8], mz, f.t[2])));
    const float B = 9.5367431640625e-07f * (fabsf(mx) + fabsf(my) + fabsf(mz) + f.c0);
    const float E = __fmaf_rn(4.0f, B, 2.384185791015625e-07f * r3);
    const float dn = (tz - f.znear) + r3;
    const float df = (f.zfar - tz) + r3;
    const float dl = __fmaf_rn(f.p2x, tx, f.p2z * tz) + r3;
    const float dr = __fmaf_rn(f.p3x, tx, f.p3z * tz) + r3;
    const float dt = __fmaf_rn(f.p4y, ty, f.p4z * tz) + r3;
    const float db = __fmaf_rn(f.p5y, ty, f.p5z * tz) + r3;
    const float m = fminf(fminf(fminf(dn, df), fminf(dl, dr)), fminf(dt, db));
    const float dz = tz - f.znear;
    zs = dz > E ? 1 : (dz < -E ? 0 : -1);
    tz_out = tz;
    return m > E ? 1 : (m < -E ? 0 : -1);
}

// ALL_LEAF: the launch covers a range known (at upload) to hold only leaves --
// the last level of a level-major tree -- so the EWA covariance is never
// needed and the kernel stays register-light (full occupancy for the
// bandwidth-bound bulk of the arena).
template <bool ALL_LEAF>
__global__ void __launch_bounds__(kMarkBlock, ALL_LEAF ? 4 : 2) k_filter_mark(const Geom g, const GeomF f,
                                                              const DevTree t,
                                                              const double tau_r,
                                                              const uint64_t begin,
                                                              const uint64_t end,
                                                              uint32_t* __restrict__ cand_bits,
                                                              uint32_t* __restrict__ qint_bits,
                                                              const uint64_t n_words) {
    // Four consecutive nodes per thread: one 16-byte load per SoA array (the
    // arrays are padded to a multiple of 256 nodes, so every float4 is aligned;
    // `begin` is a multiple of 1024).
    const uint64_t i0 = begin + (uint64_t(blockIdx.x) * kMarkBlock + threadIdx.x) * 4;
    unsigned cnib = 0, qnib = 0;
    if (i0 < end) {
        const float4 MX = __ldcs(reinterpret_cast<const float4*>(t.mx + i0));
        const float4 MY = __ldcs(reinterpret_cast<const float4*>(t.my + i0));
        const float4 MZ = __ldcs(reinterpret_cast<const float4*>(t.mz + i0));
        const float4 SX = __ldcs(reinterpret_cast<const float4*>(t.sx + i0));
        const float4 SY = __ldcs(reinterpret_cast<const float4*>(t.sy + i0));
        const float4 SZ = __ldcs(reinterpret_cast<const float4*>(t.sz + i0));
        const uint32_t LF =
            ALL_LEAF ? 0x01010101u : __ldcs(reinterpret_cast<const unsigned int*>(t.leaf + i0));
        const float mxa[4] = {MX.x, MX.y, MX.z, MX.w}, mya[4] = {MY.x, MY.y, MY.z, MY.w};
        const float mza[4] = {MZ.x, MZ.y, MZ.z, MZ.w}, sxa[4] = {SX.x, SX.y, SX.z, SX.w};
        const float sya[4] = {SY.x, SY.y, SY.z, SY.w}, sza[4] = {SZ.x, SZ.y, SZ.z, SZ.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (i0 + k >= end) break;
            const float mx = mxa[k], my = mya[k], mz = mza[k];
            const float sx = sxa[k], sy = sya[k], sz = sza[k];
            const bool leaf = ALL_LEAF || ((LF >> (8 * k)) & 0xffu) != 0;
            const float smaxf = fmaxf(fmaxf(sx, sy), sz);  // scales finite and > 0 (validated)
            float tz32;
            int zs;
            int vs = frustum_fp32(f, mx, my, mz, 3.0f * smaxf, tz32, zs);
            bool qint = false;
            if (ALL_LEAF && vs < 0) {
                double tx, ty, tz;
                cam_transform(g, mx, my, mz, tx, ty, tz);
                const double smax = std_max(std_max(double(sx), double(sy)), double(sz));
                vs = frustum_folded(g, tx, ty, tz, 3.0 * smax) ? 1 : 0;
            } else if (!ALL_LEAF && (vs < 0 || (!leaf && vs != 0))) {
                // exact FP64 path: undecided nodes, and every visible internal
                // node (its qpass needs the EWA radius, which is always FP64).
                double tx, ty, tz;
                cam_transform(g, mx, my, mz, tx, ty, tz);
                const double smax = std_max(std_max(double(sx), double(sy)), double(sz));
                vs = frustum_folded(g, tx, ty, tz, 3.0 * smax) ? 1 : 0;
                if (vs && !leaf && tz >= g.znear) {
                    const float4 q = __ldg(t.quat + i0 + k);
                    MarkOut o;
                    ewa_cov2d(g, tx, ty, tz, sx, sy, sz, q.x, q.y, q.z, q.w, o);
                    qint = o.radius <= tau_r;
                }
            }
            cnib |= (vs == 1 && (leaf || qint)) ? (1u << k) : 0u;
            qnib |= qint ? (1u << k) : 0u;
        }
    }
    // A warp covers 128 nodes = 4 words; word k gathers the nibbles of lanes 8k..8k+7.
    const unsigned lane = threadIdx.x & 31;
    unsigned cw = cnib << (4 * (lane & 7)), qw = qnib << (4 * (lane & 7));
#pragma unroll
    for (int m = 1; m < 8; m <<= 1) {
        cw |= __shfl_xor_sync(0xffffffffu, cw, m);
        qw |= __shfl_xor_sync(0xffffffffu, qw, m);
    }
    if ((lane & 7) == 0) {
        const uint64_t w = i0 >> 5;
        if (w < n_words) {
            cand_bits[w] = cw;
            qint_bits[w] = qw;
        }
    }
}

// Internal levels (the FP64-heavy 1/8 of the arena): one node per thread so
// the long covariance dependency chains of many warps overlap.
__global__ void __launch_bounds__(kMarkBlock) k_filter_mark_internal(
    const Geom g, const GeomF f, const DevTree t, const double tau_r, const uint64_t end,
    uint32_t* __restrict__ cand_bits, uint32_t* __restrict__ qint_bits, const uint64_t n_words) {
    const uint64_t i = uint64_t(blockIdx.x) * kMarkBlock + threadIdx.x;
    bool cand = false, qint = false;
    if (i < end) {
        const float mx = __ldcs(t.mx + i), my = __ldcs(t.my + i), mz = __ldcs(t.mz + i);
        const float sx = __ldcs(t.sx + i), sy = __ldcs(t.sy + i), sz = __ldcs(t.sz + i);
        const bool leaf = __ldcs(t.leaf + i) != 0;
        float tz32;
        int zs;
        int vs = frustum_fp32(f, mx, my, mz, 3.0f * fmaxf(fmaxf(sx, sy), sz), tz32, zs);
        if (vs < 0 || (!leaf && vs != 0)) {
            double tx, ty, tz;
            cam_transform(g, mx, my, mz, tx, ty, tz);
            const double smax = std_max(std_max(double(sx), double(sy)), double(sz));
            vs = frustum_folded(g, tx, ty, tz, 3.0 * smax) ? 1 : 0;
            if (vs && !leaf && tz >= g.znear) {
                const float4 q = __ldg(t.quat + i);
                MarkOut o;
                ewa_cov2d(g, tx, ty, tz, sx, sy, sz, q.x, q.y, q.z, q.w, o);
                qint = o.radius <= tau_r;
            }
        }
        cand = vs == 1 && (leaf || qint);
    }
    const unsigned cm = __ballot_sync(0xffffffffu, cand);
    const unsigned qm = __ballot_sync(0xffffffffu, qint);
    if ((threadIdx.x & 31) == 0 && (i >> 5) < n_words) {
        cand_bits[i >> 5] = cm;
        qint_bits[i >> 5] = qm;
    }
}

// K2a: candidates walk their parent chains (filter.cpp:20-25); the keep bits
// overwrite cand_bits in place (each word is read and written by one warp).
__global__ void __launch_bounds__(kSelectBlock) k_filter_select(
    uint32_t* __restrict__ cand_bits, const uint32_t* __restrict__ qint_bits,
    const uint32_t* __restrict__ parent, const uint64_t n) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t warp_base =
        uint64_t(blockIdx.x) * (kSelectBlock * kSelectItems) + uint64_t(warp) * (32 * kSelectItems);

    // All kSelectItems parent chains of a thread advance one level per round,
    // so their dependent L2 loads overlap instead of running back to back.
    uint32_t a[kSelectItems];
    bool keep[kSelectItems];
#pragma unroll
    for (int j = 0; j < kSelectItems; ++j) {
        const uint64_t node = warp_base + uint64_t(j) * 32 + lane;
        keep[j] = node < n && ((cand_bits[node >> 5] >> lane) & 1u);
        a[j] = kRootParent;
    }
#pragma unroll
    for (int j = 0; j < kSelectItems; ++j)
        if (keep[j]) a[j] = __ldg(parent + warp_base + uint64_t(j) * 32 + lane);
    while (true) {
        bool any = false;
#pragma unroll
        for (int j = 0; j < kSelectItems; ++j) any |= a[j] != kRootParent;
        if (!any) break;
        uint32_t w[kSelectItems], p[kSelectItems];
#pragma unroll
        for (int j = 0; j < kSelectItems; ++j) {
            if (a[j] != kRootParent) {
                w[j] = __ldg(qint_bits + (a[j] >> 5));
                p[j] = __ldg(parent + a[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < kSelectItems; ++j) {
            if (a[j] != kRootParent) {
                if ((w[j] >> (a[j] & 31)) & 1u) {
                    keep[j] = false;
                    a[j] = kRootParent;
                } else {
                    a[j] = p[j];
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kSelectItems; ++j) {
        const unsigned m = __ballot_sync(0xffffffffu, keep[j]);
        if (lane == 0) cand_bits[(warp_base >> 5) + j] = m;
    }
}

// K2b: ordered compaction of the keep bitmask into `selected` (strictly
// increasing, filter.cpp:147-148).  A warp owns 128 consecutive words; for
// each word (broadcast by shuffle) lane b tests bit b, so one ballot + popc
// places 32 nodes with a coalesced store.  CTA totals are chained by a
// look-back across 32,768-node tiles.
constexpr int kCompactIters = 1;  // words per lane (small tiles: one wave of short CTAs)
__global__ void __launch_bounds__(256) k_compact_bits(const uint32_t* __restrict__ bits,
                                                      const uint64_t n_words,
                                                      const uint32_t n_tiles,
                                                      uint32_t* __restrict__ selected,
                                                      unsigned long long* status,
                                                      FrameCounters* cnt) {
    __shared__ unsigned s_ticket;
    __shared__ unsigned s_warp[8];
    __shared__ unsigned long long s_excl;
    const unsigned tile = take_ticket(&cnt->ticket_select, &s_ticket);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t wbase = (uint64_t(tile) * 8 + warp) * (32 * kCompactIters);
    uint32_t words[kCompactIters];
    unsigned c = 0;
#pragma unroll
    for (int it = 0; it < kCompactIters; ++it) {
        const uint64_t w = wbase + uint64_t(it) * 32 + lane;
        words[it] = w < n_words ? __ldg(bits + w) : 0u;
        c += __popc(words[it]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if (lane == 0) s_warp[warp] = c;
    __syncthreads();
    if (warp == 0) {
        const unsigned v = lane < 8 ? s_warp[lane] : 0u;
        unsigned wi = v;
#pragma unroll
        for (int off = 1; off < 8; off <<= 1) {
            const unsigned o = __shfl_up_sync(0xffffffffu, wi, off);
            if (lane >= unsigned(off)) wi += o;
        }
        const unsigned total = __shfl_sync(0xffffffffu, wi, 7);
        if (lane < 8) s_warp[lane] = wi - v;
        const unsigned long long excl = chained_scan_warp(status, tile, total);
        if (lane == 0) {
            s_excl = excl;
            if (tile == n_tiles - 1) cnt->n_selected = excl + total;
        }
    }
    __syncthreads();
    unsigned long long pos = s_excl + s_warp[warp];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int it = 0; it < kCompactIters; ++it) {
        if (__ballot_sync(0xffffffffu, words[it] != 0u) == 0u) continue;
        for (int k = 0; k < 32; ++k) {
            const uint32_t word = __shfl_sync(0xffffffffu, words[it], k);
            if (word == 0u) continue;  // warp-uniform
            const bool bit = (word >> lane) & 1u;
            if (bit)
                selected[pos + __popc(word & lt)] =
                    uint32_t((wbase + uint64_t(it) * 32 + k) * 32 + lane);
            pos += __popc(word);
        }
    }
}

// MarkFn contract (kernels.hpp:47-52): full mark_core per node, all outputs.
__global__ void k_mark_debug(const Geom g, const DevTree t, uint64_t begin, uint64_t end,
                             double tau_r, uint8_t* vis, uint8_t* qpass, double* radius) {
    const uint64_t i = begin + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= end) return;
    const float4 q = t.quat[i];
    const MarkOut o =
        mark_core(g, t.mx[i], t.my[i], t.mz[i], t.sx[i], t.sy[i], t.sz[i], q.x, q.y, q.z, q.w, tau_r);
    vis[i - begin] = o.vis ? 1 : 0;
    qpass[i - begin] = o.qpass ? 1 : 0;
    if (radius) radius[i - begin] = o.radius;
}

void launch_filter_mark(const Geom& g, const DevTree& t, double tau_r, uint32_t* cand_bits,
                        uint32_t* qint_bits, cudaStream_t s) {
    if (t.n == 0) return;
    const GeomF f = make_geomf(g);
    const uint64_t per_cta = 4 * kMarkBlock;
    const uint64_t split = t.leaf_begin;  // multiple of per_cta; [split, n) are all leaves
    if (split > 0)
        k_filter_mark_internal<<<unsigned((split + kMarkBlock - 1) / kMarkBlock), kMarkBlock, 0, s>>>(
            g, f, t, tau_r, split, cand_bits, qint_bits, bit_words(t.n));
    if (t.n > split)
        k_filter_mark<true><<<unsigned((t.n - split + per_cta - 1) / per_cta), kMarkBlock, 0, s>>>(
            g, f, t, tau_r, split, t.n, cand_bits, qint_bits, bit_words(t.n));
}

void launch_filter_select(const DevTree& t, uint32_t* cand_bits, const uint32_t* qint_bits,
                          uint32_t* selected, unsigned long long* status, FrameCounters* cnt,
                          cudaStream_t s) {
    if (t.n == 0) return;
    k_filter_select<<<select_tiles(t.n), kSelectBlock, 0, s>>>(cand_bits, qint_bits, t.parent, t.n);
    const uint64_t n_words = bit_words(t.n);
    const uint64_t per_tile = 8ull * 32 * kCompactIters;
    const uint32_t tiles = uint32_t((n_words + per_tile - 1) / per_tile);
    k_compact_bits<<<tiles, 256, 0, s>>>(cand_bits, n_words, tiles, selected, status, cnt);
}

void launch_mark_debug(const Geom& g, const DevTree& t, uint64_t begin, uint64_t end,
                       double tau_r, uint8_t* vis, uint8_t* qpass, double* radius,
                       cudaStream_t s) {
    if (end <= begin) return;
    const unsigned grid = unsigned((end - begin + 255) / 256);
    k_mark_debug<<<grid, 256, 0, s>>>(g, t, begin, end, tau_r, vis, qpass, radius);
}

}  // namespace fgs
