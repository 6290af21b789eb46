// filter.cu -- the traversal-free parallel LoD filter (FilterGS),
// reference filter_parallel (filter.cpp:115-150).
//
// The reference marks every node (pass 1), then lets every candidate walk its
// parent chain against the marks (pass 2) and compacts the survivors in node
// order.  On the device the arena splits at `leaf_begin`: [0, leaf_begin)
// holds every internal node (1/8 of a K=8 tree), [leaf_begin, n) only leaves
// (DevTree::leaf_begin).  Three kernels per frame:
//
//   F1 k_mark_internal    [0, leaf_begin): frustum + (for visible internal
//                         nodes) the EWA radius -> cand / qint bitmasks.
//   F2 k_select_internal  [0, leaf_begin): parent-chain walks
//                         (filter.cpp:20-25) -> keep bits, compacted into
//                         `selected` in node order; the qint words are
//                         overwritten in place with blk = qint | disq, i.e.
//                         "a child of this node is disqualified".
//   F3 k_filter_leaves    [leaf_begin, n): frustum, keep = vis && !blk[parent],
//                         compacted straight into `selected` -- the leaf bulk
//                         of the arena is read exactly once and never
//                         re-visited.  The chained scan continues F2's, so
//                         `selected` comes out strictly increasing as
//                         filter.cpp:147-148 produces it.
//
// All decisions are the reference's FP64 decisions (mark_core.hpp:24-116,
// bit-exact).  They are reached in FP32 with certified error bounds, and only
// the nodes whose FP32 value falls inside the bound recompute in FP64.
#include <algorithm>
#include <cstring>
#include <cmath>

#include "launch.h"
#include "pdl.cuh"
#include "mark.cuh"
#include "scan.cuh"

namespace fgs {

// FP32 copy of the camera for the certified pre-tests.
struct GeomF {
    float r[9], t[3];
    float p2x, p2z, p3x, p3z, p4y, p4z, p5y, p5z;  // side-plane coefficients
    float znear, zfar;
    float c0;  // max(|t_i|, znear, zfar) + 1: magnitude term of the error bound
    float fx, fy;
    // qpass thresholds on lambda_max: radius = 3 sqrt(lambda) <= tau_r is
    // certain below thr_pass and impossible above thr_fail
    float thr_pass, thr_fail;
    // 4 B_max, B_max = 2^-20 (max_i |m_i|_1 + c0) over the whole tree: the
    // leaf pre-test's error term without per-node magnitude arithmetic
    float e0;
};

GeomF make_geomf(const Geom& g, double tau_r, double max_l1) {
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
    f.fx = float(g.fx);
    f.fy = float(g.fy);
    // (tau/3)^2 with a relative margin of 2^-20 each way, rounded outward to
    // float; the FP64 3*sqrt(lambda) <= tau test cannot flip inside it.
    const double l = (tau_r / 3.0) * (tau_r / 3.0);
    const double lp = l * (1.0 - 0x1p-20), lf = l * (1.0 + 0x1p-20);
    float fp = float(lp), ff = float(lf);
    if (double(fp) > lp) fp = nextafterf(fp, 0.0f);
    if (double(ff) < lf) ff = nextafterf(ff, INFINITY);
    f.thr_pass = std::isfinite(lp) ? fp : 0.0f;  // tau_r huge: no FP32 pass decision
    f.thr_fail = std::isfinite(lf) ? ff : INFINITY;
    // rounded up: f.c0 is already >= its double value + 1 - ulp; 2^-18 slack
    f.e0 = float(4.0 * 0x1p-20 * (max_l1 + double(f.c0)) * (1.0 + 0x1p-18));
    return f;
}

// Certified FP32 frustum pre-test.  With |R_ij| <= 1 and unit plane normals,
// every FP32 camera-space coordinate is within B = 2^-20 (|x|+|y|+|z|+c0) of
// the exact value (16 ulp of the magnitude sum, covering coefficient
// rounding and the three FMA roundings), and every plane distance within
// 3B + 2^-22 |.|.  When min_p(d_p + r3) clears +-E, E = 4B + 2^-22 r3, the
// FP64 reference decision (mark_core.hpp:32-40) is certain; only the
// remainder (nodes within ~1e-3 world units of a frustum plane) recompute in
// FP64.  Returns 1 visible, 0 culled, -1 undecided; zs likewise for z_ok.
struct Cam32 {
    float tx, ty, tz, B;
};
__device__ __forceinline__ int frustum_fp32(const GeomF& f, float mx, float my, float mz,
                                            float r3, Cam32& c, int& zs) {
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
    c.tx = tx;
    c.ty = ty;
    c.tz = tz;
    c.B = B;
    return m > E ? 1 : (m < -E ? 0 : -1);
}

// Leaf variant of the frustum pre-test: only vis (a leaf's z_ok and qpass are
// never read), and the magnitude term B replaced by the tree-wide bound
// B_max, so per node: transform, six plane distances, one min, and
// min_p d_p + r3 against +-(4 B_max + 2^-22 r3).  A larger B only widens the
// undecided band; decided nodes keep the reference decision.
__device__ __forceinline__ int frustum_leaf_fp32(const GeomF& f, float mx, float my, float mz,
                                                 float smax) {
    const float tx = __fmaf_rn(f.r[0], mx, __fmaf_rn(f.r[1], my, __fmaf_rn(f.r[2], mz, f.t[0])));
    const float ty = __fmaf_rn(f.r[3], mx, __fmaf_rn(f.r[4], my, __fmaf_rn(f.r[5], mz, f.t[1])));
    const float tz = __fmaf_rn(f.r[6], mx, __fmaf_rn(f.r[7], my, __fmaf_rn(f.r[8], mz, f.t[2])));
    const float r3 = 3.0f * smax;
    const float E = __fmaf_rn(2.384185791015625e-07f, r3, f.e0);
    const float dn = tz - f.znear;
    const float df = f.zfar - tz;
    const float dl = __fmaf_rn(f.p2x, tx, f.p2z * tz);
    const float dr = __fmaf_rn(f.p3x, tx, f.p3z * tz);
    const float dt = __fmaf_rn(f.p4y, ty, f.p4z * tz);
    const float db = __fmaf_rn(f.p5y, ty, f.p5z * tz);
    const float m = fminf(fminf(fminf(dn, df), fminf(dl, dr)), fminf(dt, db)) + r3;
    return m > E ? 1 : (m < -E ? 0 : -1);
}

// Certified FP32 qpass pre-test for a visible internal node with z_ok
// certain: 1 if the reference's radius = 3 sqrt(lambda_max) <= tau_r
// (mark_core.hpp:90-112), 0 if not, -1 undecided (recompute in FP64).
//
// lambda_max - 0.3 = sigma_max(M)^2 with M = J W R_q S (2x3), so the FP32
// route forms M directly (A = J W, then M = A R_q S) and bounds its error:
//   |sigma(M~) - sigma(M)| <= ||M~ - M||_F <= e,
//   e = smax * sum_i (3 dJ_i + 4 eps_R J_i),  J_i = |j_i0| + |j_i2|,
// where dJ_i bounds the error of row i of J (camera-space coordinates off by
// at most B, relative depth error rho = B / tz <= 2^-12) and eps_R = 2^-17
// bounds the FP32 rotation entries (rsqrt-normalised quaternion).  The 2x2
// Gram matrix and its closed-form top eigenvalue add at most 2^-18 (a'+c').
// e enters with a safety factor of 4; the final interval is widened by a
// further 2^-18 relative, far above the FP64 reference's own rounding
// (<= 3e-8 relative, dominated by the mid^2 - det cancellation).
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// (rcp/sqrt/rsqrt below are the approximate MUFU forms, each within 2^-22
// relative; the constants of the bound cover them.)
__device__ __forceinline__ int qpass_fp32(const GeomF& f, const Cam32& c, float sx, float sy,
                                          float sz, float4 q) {
    if (!(c.tz > 0.0f) || c.B > 2.44140625e-4f * c.tz) return -1;  // rho > 2^-12
    const float iz = rcp_approx(c.tz);
    const float rho = c.B * iz * 1.0001f;
    const float fxz = f.fx * iz, fyz = f.fy * iz;
    const float j00 = fxz, j02 = -fxz * (c.tx * iz);
    const float j11 = fyz, j12 = -fyz * (c.ty * iz);
    const float J1 = fabsf(j00) + fabsf(j02), J2 = fabsf(j11) + fabsf(j12);
    const float fB1 = fxz * iz * c.B, fB2 = fyz * iz * c.B;
    const float dJ1 = fabsf(j00) * (1.02f * rho + 1e-6f) + fabsf(j02) * (2.05f * rho + 1.5e-6f) +
                      1.02f * fB1;
    const float dJ2 = fabsf(j11) * (1.02f * rho + 1e-6f) + fabsf(j12) * (2.05f * rho + 1.5e-6f) +
                      1.02f * fB2;
    // A = J W (rows 1, 2)
    const float a0 = __fmaf_rn(j00, f.r[0], j02 * f.r[6]);
    const float a1 = __fmaf_rn(j00, f.r[1], j02 * f.r[7]);
    const float a2 = __fmaf_rn(j00, f.r[2], j02 * f.r[8]);
    const float b0 = __fmaf_rn(j11, f.r[3], j12 * f.r[6]);
    const float b1 = __fmaf_rn(j11, f.r[4], j12 * f.r[7]);
    const float b2 = __fmaf_rn(j11, f.r[5], j12 * f.r[8]);
    // R_q S (mark_core.hpp:44-60 rotation convention)
    const float n2 = __fmaf_rn(q.x, q.x, __fmaf_rn(q.y, q.y, __fmaf_rn(q.z, q.z, q.w * q.w)));
    const float inv = rsqrtf(n2);
    const float iw = q.x * inv, ix = q.y * inv, iy = q.z * inv, izq = q.w * inv;
    const float m00 = 1.0f - 2.0f * __fmaf_rn(iy, iy, izq * izq);
    const float m01 = 2.0f * __fmaf_rn(ix, iy, -(iw * izq));
    const float m02 = 2.0f * __fmaf_rn(ix, izq, iw * iy);
    const float m10 = 2.0f * __fmaf_rn(ix, iy, iw * izq);
    const float m11 = 1.0f - 2.0f * __fmaf_rn(ix, ix, izq * izq);
    const float m12 = 2.0f * __fmaf_rn(iy, izq, -(iw * ix));
    const float m20 = 2.0f * __fmaf_rn(ix, izq, -(iw * iy));
    const float m21 = 2.0f * __fmaf_rn(iy, izq, iw * ix);
    const float m22 = 1.0f - 2.0f * __fmaf_rn(ix, ix, iy * iy);
    // M = A (R_q S): column j of R_q scaled by s_j
    const float u0 = __fmaf_rn(a0, m00, __fmaf_rn(a1, m10, a2 * m20)) * sx;
    const float u1 = __fmaf_rn(a0, m01, __fmaf_rn(a1, m11, a2 * m21)) * sy;
    const float u2 = __fmaf_rn(a0, m02, __fmaf_rn(a1, m12, a2 * m22)) * sz;
    const float v0 = __fmaf_rn(b0, m00, __fmaf_rn(b1, m10, b2 * m20)) * sx;
    const float v1 = __fmaf_rn(b0, m01, __fmaf_rn(b1, m11, b2 * m21)) * sy;
    const float v2 = __fmaf_rn(b0, m02, __fmaf_rn(b1, m12, b2 * m22)) * sz;
    const float ga = __fmaf_rn(u0, u0, __fmaf_rn(u1, u1, u2 * u2));
    const float gc = __fmaf_rn(v0, v0, __fmaf_rn(v1, v1, v2 * v2));
    const float gb = __fmaf_rn(u0, v0, __fmaf_rn(u1, v1, u2 * v2));
    const float h = 0.5f * (ga - gc);
    const float s2 = 0.5f * (ga + gc) + sqrt_approx(__fmaf_rn(h, h, gb * gb));
    const float gerr = 3.814697265625e-06f * (ga + gc);  // 2^-18 (a'+c')
    const float smax = fmaxf(fmaxf(sx, sy), sz);
    const float e = 4.0f * smax * (3.0f * (dJ1 + dJ2) + 3.0517578125e-05f * (J1 + J2));
    const float sig_hi = sqrt_approx(s2 + gerr) * 1.000001f + e;
    const float sig_lo = fmaxf(sqrt_approx(fmaxf(s2 - gerr, 0.0f)) * 0.999999f - e, 0.0f);
    const float lam_hi = __fmaf_rn(sig_hi, sig_hi, 0.3f) * 1.0000039f;
    const float lam_lo = __fmaf_rn(sig_lo, sig_lo, 0.3f) * 0.9999961f;
    if (!(lam_hi == lam_hi)) return -1;  // NaN guard (validated inputs never get here)
    if (lam_hi <= f.thr_pass) return 1;
    if (lam_lo > f.thr_fail) return 0;
    return -1;
}

// Exact reference decision for one node (FP64, mark_core.hpp:27-112);
// `need_q`: the node is internal (its qpass matters).
__device__ __noinline__ void mark_fp64(const Geom& g, const DevTree& t, uint64_t i, float mx,
                                       float my, float mz, float sx, float sy, float sz,
                                       bool need_q, double tau_r, int* vis, int* qint) {
    double tx, ty, tz;
    cam_transform(g, mx, my, mz, tx, ty, tz);
    const double smax = std_max(std_max(double(sx), double(sy)), double(sz));
    const int vs = frustum_folded(g, tx, ty, tz, 3.0 * smax) ? 1 : 0;
    int qi = 0;
    if (vs && need_q && tz >= g.znear) {
        const float4 q = __ldg(t.iquat + i);
        MarkOut o;
        ewa_cov2d(g, tx, ty, tz, sx, sy, sz, q.x, q.y, q.z, q.w, o);
        qi = o.radius <= tau_r;
    }
    *vis = vs;
    *qint = qi;
}

// Exact frustum decision for leaf i (operands loaded here, so the caller keeps
// nothing live across this rarely taken call).
__device__ __noinline__ bool vis_fp64(const Geom& g, const DevTree& t, uint64_t i) {
    double tx, ty, tz;
    const float4 a = t.geo[i];
    cam_transform(g, a.x, a.y, a.z, tx, ty, tz);
    return frustum_folded(g, tx, ty, tz, 3.0 * double(a.w));
}

// Reference decision (mark_core.hpp:24-116) for node i of the internal
// region from its three records: vis, and qint = qpass && !leaf.
__device__ __forceinline__ void decide_internal(const Geom& g, const GeomF& f, const DevTree& t,
                                                uint64_t i, float4 a, float4 sc, float4 q,
                                                double tau_r, bool& vis, bool& qint) {
    const bool leaf = sc.w != 0.0f;
    Cam32 c;
    int zs;
    int vs = frustum_fp32(f, a.x, a.y, a.z, 3.0f * a.w, c, zs);
    int qs = 0;
    if (vs == 1 && !leaf) {
        if (zs == 1) qs = qpass_fp32(f, c, sc.x, sc.y, sc.z, q);
        else if (zs < 0) qs = -1;  // zs == 0: z_ok false, qpass false for certain
    }
    if (vs < 0 || qs < 0) {
        int v, qi;
        mark_fp64(g, t, i, a.x, a.y, a.z, sc.x, sc.y, sc.z, !leaf, tau_r, &v, &qi);
        vs = v;
        qs = qi;
    }
    vis = vs == 1;
    qint = vs == 1 && qs == 1;
}

// F1: internal region [0, leaf_begin).  Persistent grid; each warp walks
// 32-node groups (one node per lane) and issues the three 16-byte records of
// its next group (mean + max scale, scales + leaf flag, quaternion) before
// evaluating the current one, so loads overlap the FP32 EWA arithmetic:
// frustum, and for visible internal nodes the radius -> cand / qint words by
// ballot.
#ifndef MARK_MIN_CTAS
#define MARK_MIN_CTAS 3
#endif
__global__ void __launch_bounds__(kMarkBlock, MARK_MIN_CTAS) k_mark_internal(
    const __grid_constant__ Geom g, const GeomF f, const __grid_constant__ DevTree t,
    const double tau_r, uint32_t* __restrict__ cand_bits, uint32_t* __restrict__ qint_bits,
    FilterClock* clk) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    clock_start(clk, 0);
    const unsigned lane = threadIdx.x & 31;
    const uint64_t end = t.leaf_begin;
    const uint64_t n_groups = (end + 31) / 32;
    const uint64_t stride = uint64_t(gridDim.x) * (kMarkBlock / 32);
    uint64_t grp = uint64_t(blockIdx.x) * (kMarkBlock / 32) + (threadIdx.x >> 5);
    float4 a, sc, q;
    auto load = [&](uint64_t gi) {
        const uint64_t i = gi * 32 + lane;
        if (gi < n_groups && i < end) {
            a = __ldcs(t.geo + i);
            sc = __ldcs(t.iscale + i);
            q = __ldcs(t.iquat + i);
        }
    };
    load(grp);
    for (; grp < n_groups; grp += stride) {
        const uint64_t i = grp * 32 + lane;
        const float4 ca = a, csc = sc, cq = q;
        load(grp + stride);
        bool cand = false, qint = false;
        if (i < end) {
            bool vis;
            decide_internal(g, f, t, i, ca, csc, cq, tau_r, vis, qint);
            cand = vis && (csc.w != 0.0f || qint);
        }
        const unsigned cm = __ballot_sync(0xffffffffu, cand);
        const unsigned qm = __ballot_sync(0xffffffffu, qint);
        if (lane == 0) {
            cand_bits[grp] = cm;
            qint_bits[grp] = qm;
        }
    }
    clock_end(clk, 0);
}

// Survivor counts are kept per 8192-node tile (one count per k_compact CTA).
// A compaction CTA's output position is the sum of the preceding tiles' counts:
// summed directly by the CTA up to kDirectPrefixTiles tiles (cfg 3: 1,226), and
// above that (cfg 4: 6,121 tiles, where the direct sums are O(T^2) = 18.7M loads)
// scanned once by k_tile_prefix between F3 and F4.
constexpr int kTileNodes = 8192;
constexpr uint64_t kDirectPrefixTiles = 2048;
__host__ __device__ inline uint64_t count_tiles(uint64_t n) {
    return (n + kTileNodes - 1) / kTileNodes;
}
__device__ __forceinline__ void count_survivors(uint32_t* tile_count, uint64_t tile, uint32_t c) {
    atomicAdd(tile_count + tile, c);
}

// F2: internal region.  Every node walks its parent chain (filter.cpp:20-25)
// against the qint bitmask (L2-resident: 1 bit per internal node); the
// kSelectItems chains of a thread advance one level per round so their
// dependent loads overlap.  keep = cand && !disq replaces the cand word; the
// qint word is replaced by blk = qint | disq ("a child of this node is
// disqualified").  Another warp may read either value of a qint word while
// walking: for any descendant the OR along its chain is the same, so the
// result does not depend on the interleaving.
__device__ __forceinline__ void select_body(uint32_t* __restrict__ cand_bits, uint32_t* qint_bits,
                                            const uint32_t* __restrict__ parent, const uint64_t end,
                                            uint32_t* __restrict__ tile_count, const unsigned block) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t warp_base =
        uint64_t(block) * (kSelectBlock * kSelectItems) + uint64_t(warp) * (32 * kSelectItems);
    if (warp_base >= end) return;  // warp-uniform
    uint32_t a[kSelectItems];
    bool disq[kSelectItems];
#pragma unroll
    for (int j = 0; j < kSelectItems; ++j) {
        a[j] = __ldg(parent + warp_base + uint64_t(j) * 32 + lane);
        disq[j] = false;
    }
    while (true) {
        bool any = false;
#pragma unroll
        for (int j = 0; j < kSelectItems; ++j) any |= a[j] != kRootParent;
        if (!any) break;
        uint32_t w[kSelectItems], p[kSelectItems];
#pragma unroll
        for (int j = 0; j < kSelectItems; ++j) {
            if (a[j] != kRootParent) {
                w[j] = *(volatile const uint32_t*)(qint_bits + (a[j] >> 5));
                p[j] = __ldg(parent + a[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < kSelectItems; ++j) {
            if (a[j] != kRootParent) {
                if ((w[j] >> (a[j] & 31)) & 1u) {
                    disq[j] = true;
                    a[j] = kRootParent;
                } else {
                    a[j] = p[j];
                }
            }
        }
    }
    uint32_t mine = 0;  // lane j < kSelectItems takes word j
#pragma unroll
    for (int j = 0; j < kSelectItems; ++j) {
        const uint32_t dm = __ballot_sync(0xffffffffu, disq[j]);
        if (lane == unsigned(j)) mine = dm;
    }
    const uint64_t wi = (warp_base >> 5) + lane;
    unsigned cntw = 0;
    if (lane < unsigned(kSelectItems) && wi * 32 < end) {
        const uint32_t keep = cand_bits[wi] & ~mine;
        cand_bits[wi] = keep;
        if (mine) qint_bits[wi] |= mine;
        cntw = __popc(keep);
    }
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) cntw += __shfl_xor_sync(0xffffffffu, cntw, off);
    if (lane == 0 && cntw) count_survivors(tile_count, warp_base / kTileNodes, cntw);
}

#ifndef SELECT_LB
#define SELECT_LB 0
#endif
#if SELECT_LB
__global__ void __launch_bounds__(kSelectBlock, SELECT_LB) k_select_internal(
#else
__global__ void __launch_bounds__(kSelectBlock) k_select_internal(
#endif
    uint32_t* __restrict__ cand_bits, uint32_t* qint_bits, const uint32_t* __restrict__ parent,
    const uint64_t end, uint32_t* __restrict__ tile_count, FilterClock* clk) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    clock_start(clk, 1);
    select_body(cand_bits, qint_bits, parent, end, tile_count, blockIdx.x);
    clock_end(clk, 1);
}

// F3: the all-leaf suffix [leaf_begin, n).  A leaf is kept iff visible
// (filter.cpp:137; a leaf's qpass is never read) and no ancestor is
// disqualifying, i.e. its parent's blk bit (F2) is clear.  The blk test comes
// first: it needs only the parent index, and a leaf under a blocked parent is
// dropped whatever its frustum test says, so its 16-byte geo record is never
// fetched (siblings are contiguous, so whole sectors are skipped).  Warp =
// 128 consecutive leaves, lane l taking leaves l, l+32, l+64, l+96: every
// parent load is one contiguous 128 B warp access (arrays padded to a
// multiple of 256 nodes; leaf_begin a multiple of 1024).  Writes keep words
// (one ballot each) and the per-tile survivor counts.
#ifndef LEAF_PER_LANE
#define LEAF_PER_LANE 4
#endif
constexpr int kLeafPerLane = LEAF_PER_LANE;  // leaves per lane (a warp: 32 kLeafPerLane)
// F3 (and its multi-view form) budgeted for 8 CTAs per SM (32 registers): the leaf pass
// is a dependent load chain, occupancy hides it (leaves + compaction 31.5 -> 30.4 us per
// frame; F2 likewise at 8 CTAs was slower, 28.4 -> 31.9 us)
#ifndef LEAF_LB
#define LEAF_LB 8
#endif
#if LEAF_LB
__global__ void __launch_bounds__(256, LEAF_LB) k_filter_leaves(
#else
__global__ void __launch_bounds__(256) k_filter_leaves(
#endif
    const __grid_constant__ Geom g, const GeomF f, const __grid_constant__ DevTree t,
    const uint32_t* __restrict__ blk_bits, uint32_t* __restrict__ keep_bits,
    uint32_t* __restrict__ tile_count, FilterClock* clk) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    clock_start(clk, 2);
    const unsigned lane = threadIdx.x & 31;
    const uint64_t end = t.n;
    const uint64_t wbase =
        t.leaf_begin + (uint64_t(blockIdx.x) * 256 + (threadIdx.x & ~31u)) * kLeafPerLane;
    if (wbase >= end) return;  // warp-uniform
    uint32_t p[kLeafPerLane];
#pragma unroll
    for (int k = 0; k < kLeafPerLane; ++k) p[k] = __ldcs(t.parent + wbase + k * 32 + lane);
    unsigned need = 0;
#pragma unroll
    for (int k = 0; k < kLeafPerLane; ++k) {
        const bool in = wbase + k * 32 + lane < end;  // padding past n never survives
        const bool blocked =
            p[k] != kRootParent && ((__ldg(blk_bits + (p[k] >> 5)) >> (p[k] & 31)) & 1u);
        need |= (in && !blocked) ? (1u << k) : 0u;
    }
    float4 a[kLeafPerLane];
#pragma unroll
    for (int k = 0; k < kLeafPerLane; ++k)
        if ((need >> k) & 1u) a[k] = __ldcs(t.geo + wbase + k * 32 + lane);
    unsigned keep = 0, undec = 0;
#pragma unroll
    for (int k = 0; k < kLeafPerLane; ++k) {
        if ((need >> k) & 1u) {
            const int vs = frustum_leaf_fp32(f, a[k].x, a[k].y, a[k].z, a[k].w);
            keep |= vs == 1 ? (1u << k) : 0u;
            undec |= vs < 0 ? (1u << k) : 0u;
        }
    }
    if (undec) {
        // rare: within ~1e-3 world units of a frustum plane -> exact FP64
        // decision; operands re-read so nothing stays live across the call
        for (int k = 0; k < kLeafPerLane; ++k)
            if ((undec >> k) & 1u) keep |= vis_fp64(g, t, wbase + k * 32 + lane) ? (1u << k) : 0u;
    }
    unsigned c = 0;
#pragma unroll
    for (int k = 0; k < kLeafPerLane; ++k) {
        const uint32_t w = __ballot_sync(0xffffffffu, (keep >> k) & 1u);
        if (lane == unsigned(k) && (wbase + k * 32) < end) keep_bits[(wbase >> 5) + k] = w;
        c += __popc(w);
    }
    // a warp's 128 leaves lie in one 8192-node tile (leaf_begin is a multiple of 1024)
    if (lane == 0 && c) count_survivors(tile_count, wbase / kTileNodes, c);
    clock_end(clk, 2);
}

// Exclusive scan of the per-tile survivor counts (large trees only): one CTA,
// thread k owning a contiguous run of tiles.
__global__ void __launch_bounds__(1024) k_tile_prefix(const uint32_t* __restrict__ tile_count,
                                                      const uint32_t n_tiles,
                                                      uint32_t* __restrict__ prefix) {
    pdl_wait();
    pdl_trigger();
    __shared__ uint32_t s_warp[32];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t per = (n_tiles + 1023) / 1024;
    const uint32_t t0 = min(n_tiles, threadIdx.x * per), t1 = min(n_tiles, t0 + per);
    uint32_t sum = 0;
    for (uint32_t t = t0; t < t1; ++t) sum += tile_count[t];
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= unsigned(o)) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t v = s_warp[lane];
        uint32_t wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= unsigned(o)) wi += u;
        }
        s_warp[lane] = wi - v;  // exclusive over warps
    }
    __syncthreads();
    uint32_t run = s_warp[warp] + (incl - sum);
    for (uint32_t t = t0; t < t1; ++t) {
        prefix[t] = run;
        run += tile_count[t];
    }
}

// F4: ordered compaction of the keep words into `selected` (strictly
// increasing, filter.cpp:147-148).  One CTA per 8192-node tile; its first
// output position is the sum of the counts of all preceding tiles (read
// directly: no look-back chain, CTAs never wait on each other).  Warp w owns
// 32 words; for every non-empty word (broadcast by shuffle) lane b tests bit
// b, so one popc places 32 nodes with a coalesced store.
__device__ __forceinline__ void compact_body(const uint32_t* __restrict__ keep_bits,
                                             const uint64_t n_words,
                                             const uint32_t* __restrict__ tile_count,
                                             uint32_t* __restrict__ selected, FrameCounters* cnt,
                                             const uint32_t* __restrict__ prefix,
                                             const unsigned tile, const unsigned n_tiles) {
    __shared__ unsigned s_red[8];
    __shared__ unsigned s_warp[8];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // survivors before this tile: scanned by k_tile_prefix, or summed here
    unsigned pre = 0;
    if (prefix) {
        if (threadIdx.x == 0) pre = __ldg(prefix + tile);
    } else {
        unsigned p4[4] = {0u, 0u, 0u, 0u};
        unsigned k = threadIdx.x;
        for (; k + 768 < tile; k += 1024) {
#pragma unroll
            for (int u = 0; u < 4; ++u) p4[u] += __ldg(tile_count + k + 256 * u);
        }
        for (; k < tile; k += 256) p4[0] += __ldg(tile_count + k);
        pre = (p4[0] + p4[1]) + (p4[2] + p4[3]);
    }
    const uint64_t wi = uint64_t(tile) * (kTileNodes / 32) + warp * 32 + lane;
    const uint32_t keepw = wi < n_words ? __ldg(keep_bits + wi) : 0u;
    unsigned c = __popc(keepw);
    unsigned incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= unsigned(off)) incl += o;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, off);
    if (lane == 31) s_warp[warp] = incl;
    if (lane == 0) s_red[warp] = pre;
    __syncthreads();
    unsigned base = 0, before = 0, total = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        base += s_red[k];
        before += k < int(warp) ? s_warp[k] : 0u;
        total += s_warp[k];
    }
    if (tile == n_tiles - 1 && threadIdx.x == 0) cnt->n_selected = uint64_t(base) + total;
    const unsigned long long pos = uint64_t(base) + before;
    const unsigned lt = (1u << lane) - 1u;
    unsigned nz = __ballot_sync(0xffffffffu, keepw != 0u);
    const uint64_t warp_node = (uint64_t(tile) * (kTileNodes / 32) + warp * 32) * 32;
    while (nz) {  // non-empty words only (warp-uniform)
        const int j = __ffs(nz) - 1;
        nz &= nz - 1;
        const uint32_t word = __shfl_sync(0xffffffffu, keepw, j);
        const unsigned at = __shfl_sync(0xffffffffu, incl, j) - __popc(word);
        if ((word >> lane) & 1u)
            selected[pos + at + __popc(word & lt)] = uint32_t(warp_node + uint64_t(j) * 32 + lane);
    }
}

__global__ void __launch_bounds__(256) k_compact(const uint32_t* __restrict__ keep_bits,
                                                 const uint64_t n_words,
                                                 const uint32_t* __restrict__ tile_count,
                                                 uint32_t* __restrict__ selected,
                                                 FrameCounters* cnt, FilterClock* clk,
                                                 const int clock_slot,
                                                 const uint32_t* __restrict__ prefix) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    clock_start(clk, clock_slot);
    compact_body(keep_bits, n_words, tile_count, selected, cnt, prefix, blockIdx.x, gridDim.x);
    clock_end(clk, clock_slot);
}

// ---- serial (level-wise) filter, reference filter_serial (filter.cpp:60-113) --
// The ablation baseline of the paper's Table 2:
// one kernel and one barrier per level.  Level l is processed flat over its
// node range: a node is active iff l == 0 or its parent was expanded (visible,
// not qpass, not a leaf); an active visible node is selected if qpass or leaf
// and expanded otherwise -- exactly the reference's active-list recursion,
// kept as bitmasks so `selected` comes out in node order (the reference's
// level-major, parent-ordered output is ascending, test_filter.cpp:126).
// Words straddling a level boundary are merged with atomicOr (both bitmasks
// are cleared first).  level_flag[l] != 0 iff level l had an active node.
__global__ void __launch_bounds__(256) k_serial_level(
    const __grid_constant__ Geom g, const GeomF f, const __grid_constant__ DevTree t,
    const double tau_r, const uint64_t b, const uint64_t e, const int level,
    uint32_t* __restrict__ sel_bits, uint32_t* __restrict__ exp_bits,
    uint32_t* __restrict__ tile_count, unsigned* level_flag, FrameCounters* cnt,
    FilterClock* clk) {
    const int slot = level < kFilterClocks - 1 ? level : kFilterClocks - 2;
    clock_start(clk, slot);
    const unsigned lane = threadIdx.x & 31;
    const uint64_t i = (b & ~uint64_t(31)) + uint64_t(blockIdx.x) * 256 + threadIdx.x;
    bool sel = false, expand = false, active = false;
    if (i >= b && i < e) {
        const uint32_t p = t.parent[i];
        active = level == 0 || (p != kRootParent && ((exp_bits[p >> 5] >> (p & 31)) & 1u));
        if (active) {
            const float4 a = t.geo[i];
            if (i < t.leaf_begin) {
                bool vis, qint;
                decide_internal(g, f, t, i, a, t.iscale[i], t.iquat[i], tau_r, vis, qint);
                const bool leaf = t.iscale[i].w != 0.0f;
                sel = vis && (qint || leaf);
                expand = vis && !qint && !leaf;
            } else {  // all-leaf suffix: only vis matters
                int vs = frustum_leaf_fp32(f, a.x, a.y, a.z, a.w);
                if (vs < 0) vs = vis_fp64(g, t, i) ? 1 : 0;
                sel = vs == 1;
            }
        }
    }
    const unsigned sm = __ballot_sync(0xffffffffu, sel);
    const unsigned em = __ballot_sync(0xffffffffu, expand);
    const unsigned am = __ballot_sync(0xffffffffu, active);
    if (lane == 0) {
        const uint64_t w = i >> 5;
        const bool whole = (w << 5) >= b && ((w + 1) << 5) <= e;
        if (whole) {
            sel_bits[w] = sm;
            exp_bits[w] = em;
        } else {
            if (sm) atomicOr(sel_bits + w, sm);
            if (em) atomicOr(exp_bits + w, em);
        }
        if (sm) count_survivors(tile_count, i / kTileNodes, __popc(sm));
        if (am && !level_flag[level] && atomicOr(level_flag + level, 1u) == 0u)
            atomicAdd(&cnt->serial_passes, 1u);
    }
    clock_end(clk, slot);
}

void launch_filter_serial(const Geom& g, const DevTree& t, double tau_r,
                          const uint64_t* level_begin, int n_levels, uint32_t* sel_bits,
                          uint32_t* exp_bits, uint32_t* tile_count, unsigned* level_flag,
                          uint32_t* selected, FrameCounters* cnt, cudaEvent_t* level_events,
                          cudaStream_t s, FilterClock* clk) {
    if (t.n == 0) return;
    const GeomF f = make_geomf(g, tau_r, t.max_l1);
    cudaMemsetAsync(sel_bits, 0, ((t.n + 31) / 32) * 4, s);
    cudaMemsetAsync(exp_bits, 0, ((t.n + 31) / 32) * 4, s);
    for (int l = 0; l < n_levels; ++l) {
        const uint64_t b = level_begin[l], e = l + 1 < n_levels ? level_begin[l + 1] : t.n;
        if (level_events) cudaEventRecord(level_events[l], s);
        if (e <= b) continue;
        const uint64_t span = e - (b & ~uint64_t(31));
        k_serial_level<<<unsigned((span + 255) / 256), 256, 0, s>>>(
            g, f, t, tau_r, b, e, l, sel_bits, exp_bits, tile_count, level_flag, cnt, clk);
    }
    if (level_events) cudaEventRecord(level_events[n_levels], s);
    const uint64_t T = count_tiles(t.n);
    uint32_t* prefix = T > kDirectPrefixTiles ? tile_count + T : nullptr;
    if (prefix) k_tile_prefix<<<1, 1024, 0, s>>>(tile_count, uint32_t(T), prefix);
    k_compact<<<unsigned(T), 256, 0, s>>>(sel_bits, (t.n + 31) / 32, tile_count, selected, cnt,
                                          clk, kFilterClocks - 1, prefix);
}

// MarkFn contract (kernels.hpp:47-52): full mark_core per node, all outputs.
__global__ void k_mark_debug(const Geom g, const DevTree t, uint64_t begin, uint64_t end,
                             double tau_r, uint8_t* vis, uint8_t* qpass, double* radius) {
    const uint64_t i = begin + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= end) return;
    const SplatRec r = t.splat[i];
    const MarkOut o =
        mark_core(g, r.mx, r.my, r.mz, r.sx, r.sy, r.sz, r.qw, r.qx, r.qy, r.qz, tau_r);
    vis[i - begin] = o.vis ? 1 : 0;
    qpass[i - begin] = o.qpass ? 1 : 0;
    if (radius) radius[i - begin] = o.radius;
}

// SMs of the current device (persistent grids), cached per device.
static int sm_count() {
    static int cache[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 148;
    }
    return cache[dev];
}

uint32_t filter_status_entries(uint64_t n) {
    const uint64_t t = count_tiles(n);
    return uint32_t(2 * t + 1);  // counts, then (large trees) their exclusive prefix
}

int filter_launches(uint64_t n) { return count_tiles(n) > kDirectPrefixTiles ? 5 : 4; }

void launch_filter(const Geom& g, const DevTree& t, double tau_r, uint32_t* cand_bits,
                   uint32_t* qint_bits, uint32_t* tile_count, uint32_t* selected,
                   FrameCounters* cnt, cudaStream_t s, cudaEvent_t mid, FilterClock* clk) {
    if (t.n == 0) {
        if (mid) cudaEventRecord(mid, s);
        return;
    }
    const GeomF f = make_geomf(g, tau_r, t.max_l1);
    const uint64_t split = t.leaf_begin;  // [split, n) are all leaves
    if (split > 0) {
        const uint64_t groups = (split + 31) / 32;
        const unsigned grid =
            unsigned(std::min<uint64_t>((groups + 7) / 8, uint64_t(sm_count()) * MARK_MIN_CTAS));
        launch_pdl(k_mark_internal, grid, kMarkBlock, 0, s, g, f, t, tau_r, cand_bits, qint_bits,
                   clk);
        const uint64_t per = uint64_t(kSelectBlock) * kSelectItems;
        launch_pdl(k_select_internal, unsigned((split + per - 1) / per), kSelectBlock, 0, s,
                   cand_bits, qint_bits, t.parent, split, tile_count, clk);
    }
    if (mid) cudaEventRecord(mid, s);
    if (t.n > split) {
        const uint64_t per_cta = 256ull * kLeafPerLane;
        launch_pdl(k_filter_leaves, unsigned((t.n - split + per_cta - 1) / per_cta), 256, 0, s, g,
                   f, t, static_cast<const uint32_t*>(qint_bits), cand_bits, tile_count, clk);
    }
    const uint64_t T = count_tiles(t.n);
    uint32_t* prefix = T > kDirectPrefixTiles ? tile_count + T : nullptr;
    if (prefix)
        launch_pdl(k_tile_prefix, 1, 1024, 0, s, static_cast<const uint32_t*>(tile_count),
                   uint32_t(T), prefix);
    launch_pdl(k_compact, unsigned(T), 256, 0, s, static_cast<const uint32_t*>(cand_bits),
               (t.n + 31) / 32, static_cast<const uint32_t*>(tile_count), selected, cnt, clk, 3,
               static_cast<const uint32_t*>(prefix));
}

// ---- multi-view filter (SURVEY 8(e)'s option: several views per pass) ----
// One pass over the node arrays serves up to kMaxViews views of the same tree:
// F1 loads each internal node's three records once and decides it for every
// view; F3 loads each leaf's parent index once, tests the blk bit of every view
// and fetches the geo record once if any view needs it.  F2 and F4 run per view
// (blockIdx.y) with their single-view code.  Every output is the single-view
// filter's, bit for bit (each view's decisions are the same FP32 / FP64 code).
struct ViewSetDev {
    Geom g[kMaxViews];
    GeomF f[kMaxViews];
    uint32_t* cand[kMaxViews];
    uint32_t* qint[kMaxViews];
    uint32_t* tile_count[kMaxViews];  // survivor counts, then (large trees) their prefix
    uint32_t* selected[kMaxViews];
    FrameCounters* cnt[kMaxViews];
    int n;
};

#ifndef MARK_VIEWS_MIN_CTAS
#define MARK_VIEWS_MIN_CTAS MARK_MIN_CTAS
#endif
__global__ void __launch_bounds__(kMarkBlock, MARK_VIEWS_MIN_CTAS) k_mark_views(
    const __grid_constant__ ViewSetDev vs, const __grid_constant__ DevTree t, const double tau_r) {
    pdl_wait();
    pdl_trigger();
    const unsigned lane = threadIdx.x & 31;
    const uint64_t end = t.leaf_begin;
    const uint64_t n_groups = (end + 31) / 32;
    const uint64_t stride = uint64_t(gridDim.x) * (kMarkBlock / 32);
    uint64_t grp = uint64_t(blockIdx.x) * (kMarkBlock / 32) + (threadIdx.x >> 5);
    float4 a, sc, q;
    auto load = [&](uint64_t gi) {
        const uint64_t i = gi * 32 + lane;
        if (gi < n_groups && i < end) {
            a = __ldcs(t.geo + i);
            sc = __ldcs(t.iscale + i);
            q = __ldcs(t.iquat + i);
        }
    };
    load(grp);
    for (; grp < n_groups; grp += stride) {
        const uint64_t i = grp * 32 + lane;
        const float4 ca = a, csc = sc, cq = q;
        load(grp + stride);
#pragma unroll 1
        for (int v = 0; v < vs.n; ++v) {
            bool cand = false, qint = false;
            if (i < end) {
                bool vis;
                decide_internal(vs.g[v], vs.f[v], t, i, ca, csc, cq, tau_r, vis, qint);
                cand = vis && (csc.w != 0.0f || qint);
            }
            const unsigned cm = __ballot_sync(0xffffffffu, cand);
            const unsigned qm = __ballot_sync(0xffffffffu, qint);
            if (lane == 0) {
                vs.cand[v][grp] = cm;
                vs.qint[v][grp] = qm;
            }
        }
    }
}

__global__ void __launch_bounds__(kSelectBlock) k_select_views(const __grid_constant__ ViewSetDev vs,
                                                               const uint32_t* __restrict__ parent,
                                                               const uint64_t end) {
    pdl_wait();
    pdl_trigger();
    const int v = int(blockIdx.y);
    select_body(vs.cand[v], vs.qint[v], parent, end, vs.tile_count[v], blockIdx.x);
}

// the multi-view leaf pass measured alike at 4 / 6 / 8 CTAs per SM (64 / 40 / 32
// registers; 6 and 8 spill): 4
#ifndef LEAF_VIEWS_LB
#define LEAF_VIEWS_LB 4
#endif
__global__ void __launch_bounds__(256, LEAF_VIEWS_LB) k_leaves_views(const __grid_constant__ ViewSetDev vs,
                                                      const __grid_constant__ DevTree t) {
    pdl_wait();
    pdl_trigger();
    const unsigned lane = threadIdx.x & 31;
    const uint64_t end = t.n;
    const uint64_t wbase =
        t.leaf_begin + (uint64_t(blockIdx.x) * 256 + (threadIdx.x & ~31u)) * kLeafPerLane;
    if (wbase >= end) return;  // warp-uniform
    uint32_t p[kLeafPerLane];
#pragma unroll
    for (int k = 0; k < kLeafPerLane; ++k) p[k] = __ldcs(t.parent + wbase + k * 32 + lane);
    unsigned need[kMaxViews], any = 0;
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v) {
        need[v] = 0;
        if (v < vs.n) {
#pragma unroll
            for (int k = 0; k < kLeafPerLane; ++k) {
                const bool in = wbase + k * 32 + lane < end;
                const bool blocked = p[k] != kRootParent &&
                                     ((__ldg(vs.qint[v] + (p[k] >> 5)) >> (p[k] & 31)) & 1u);
                need[v] |= (in && !blocked) ? (1u << k) : 0u;
            }
            any |= need[v];
        }
    }
    float4 a[kLeafPerLane];
#pragma unroll
    for (int k = 0; k < kLeafPerLane; ++k)
        if ((any >> k) & 1u) a[k] = __ldcs(t.geo + wbase + k * 32 + lane);
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v) {
        if (v >= vs.n) break;
        unsigned keep = 0, undec = 0;
#pragma unroll
        for (int k = 0; k < kLeafPerLane; ++k) {
            if ((need[v] >> k) & 1u) {
                const int r = frustum_leaf_fp32(vs.f[v], a[k].x, a[k].y, a[k].z, a[k].w);
                keep |= r == 1 ? (1u << k) : 0u;
                undec |= r < 0 ? (1u << k) : 0u;
            }
        }
        if (undec) {
            for (int k = 0; k < kLeafPerLane; ++k)
                if ((undec >> k) & 1u)
                    keep |= vis_fp64(vs.g[v], t, wbase + k * 32 + lane) ? (1u << k) : 0u;
        }
        unsigned c = 0;
#pragma unroll
        for (int k = 0; k < kLeafPerLane; ++k) {
            const uint32_t w = __ballot_sync(0xffffffffu, (keep >> k) & 1u);
            if (lane == unsigned(k) && (wbase + k * 32) < end) vs.cand[v][(wbase >> 5) + k] = w;
            c += __popc(w);
        }
        if (lane == 0 && c) count_survivors(vs.tile_count[v], wbase / kTileNodes, c);
    }
}

__global__ void __launch_bounds__(1024) k_tile_prefix_views(const __grid_constant__ ViewSetDev vs,
                                                            const uint32_t n_tiles) {
    // k_tile_prefix's scan for view blockIdx.y (large trees only)
    pdl_wait();
    pdl_trigger();
    const uint32_t* tile_count = vs.tile_count[blockIdx.y];
    uint32_t* prefix = vs.tile_count[blockIdx.y] + n_tiles;
    __shared__ uint32_t s_warp[32];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t per = (n_tiles + 1023) / 1024;
    const uint32_t t0 = min(n_tiles, threadIdx.x * per), t1 = min(n_tiles, t0 + per);
    uint32_t sum = 0;
    for (uint32_t t = t0; t < t1; ++t) sum += tile_count[t];
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= unsigned(o)) incl += u;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t u = s_warp[lane];
        uint32_t wi = u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= unsigned(o)) wi += x;
        }
        s_warp[lane] = wi - u;
    }
    __syncthreads();
    uint32_t run = s_warp[warp] + (incl - sum);
    for (uint32_t t = t0; t < t1; ++t) {
        prefix[t] = run;
        run += tile_count[t];
    }
}

__global__ void __launch_bounds__(256) k_compact_views(const __grid_constant__ ViewSetDev vs,
                                                       const uint64_t n_words,
                                                       const int with_prefix) {
    pdl_wait();
    pdl_trigger();
    const int v = int(blockIdx.y);
    compact_body(vs.cand[v], n_words, vs.tile_count[v], vs.selected[v], vs.cnt[v],
                 with_prefix ? vs.tile_count[v] + gridDim.x : nullptr, blockIdx.x, gridDim.x);
}

void launch_filter_views(const ViewSet& views, const DevTree& t, double tau_r, cudaStream_t s) {
    if (views.n <= 0 || t.n == 0) return;
    ViewSetDev vs;
    std::memset(&vs, 0, sizeof(vs));
    vs.n = views.n;
    for (int v = 0; v < views.n; ++v) {
        vs.g[v] = views.g[v];
        vs.f[v] = make_geomf(views.g[v], tau_r, t.max_l1);
        vs.cand[v] = views.cand[v];
        vs.qint[v] = views.qint[v];
        vs.tile_count[v] = views.tile_count[v];
        vs.selected[v] = views.selected[v];
        vs.cnt[v] = views.cnt[v];
    }
    const uint64_t split = t.leaf_begin;
    if (split > 0) {
        const uint64_t groups = (split + 31) / 32;
        const unsigned grid =
            unsigned(std::min<uint64_t>((groups + 7) / 8, uint64_t(sm_count()) * MARK_MIN_CTAS));
        const unsigned vgrid = unsigned(
            std::min<uint64_t>((groups + 7) / 8, uint64_t(sm_count()) * MARK_VIEWS_MIN_CTAS));
        launch_pdl(k_mark_views, vgrid, kMarkBlock, 0, s, vs, t, tau_r);
        const uint64_t per = uint64_t(kSelectBlock) * kSelectItems;
        launch_pdl(k_select_views, dim3(unsigned((split + per - 1) / per), unsigned(views.n)),
                   kSelectBlock, 0, s, vs, static_cast<const uint32_t*>(t.parent), split);
    }
    if (t.n > split) {
        const uint64_t per_cta = 256ull * kLeafPerLane;
        launch_pdl(k_leaves_views, unsigned((t.n - split + per_cta - 1) / per_cta), 256, 0, s, vs,
                   t);
    }
    const uint64_t T = count_tiles(t.n);
    const int with_prefix = T > kDirectPrefixTiles ? 1 : 0;
    if (with_prefix)
        launch_pdl(k_tile_prefix_views, dim3(1, unsigned(views.n)), 1024, 0, s, vs, uint32_t(T));
    launch_pdl(k_compact_views, dim3(unsigned(T), unsigned(views.n)), 256, 0, s, vs,
               (t.n + 31) / 32, with_prefix);
}

void launch_mark_debug(const Geom& g, const DevTree& t, uint64_t begin, uint64_t end,
                       double tau_r, uint8_t* vis, uint8_t* qpass, double* radius,
                       cudaStream_t s) {
    if (end <= begin) return;
    const unsigned grid = unsigned((end - begin + 255) / 256);
    k_mark_debug<<<grid, 256, 0, s>>>(g, t, begin, end, tau_r, vis, qpass, radius);
}

}  // namespace fgs
