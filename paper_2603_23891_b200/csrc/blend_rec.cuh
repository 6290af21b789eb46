// blend_rec.cuh -- the per-pair blend record of the TMA-staged blend (K6).
//
// Written at the pair's sorted position, so each tile's records are one
// contiguous, blend-ordered range that k_blend_tma streams into shared memory
// with cp.async.bulk.  The sort kernels write it where they place each key
// (sort.cu); k_pack_blend writes it in a separate pass for sorted keys that
// come from elsewhere (stage entry points).
#pragma once

#include "common.cuh"

namespace fgs {

struct __align__(16) BlendRec {
    float4 geo;  // tile-relative mean x, y, ha, hc
    float4 ct;   // cb, ethr, op, r
    float4 gbm;  // g, b, block mask (bits), slot (bits)
};
static_assert(sizeof(BlendRec) == 48, "bulk copies move whole 16-byte-aligned records");

// Where and how a sort kernel emits the records of one tile's bucket.
struct RecOut {
    BlendRec* rec;  // null: keys only
    const Gauss64* g64;
    const Gauss32* g32;
};

#ifdef __CUDACC__
// The record of slot gi in the tile whose pixel origin is (tx0, ty0): the
// tile-relative mean rounded once from FP64 (as the warp-block means of
// k_blend_ws were), and the 8-bit mask of the tile's 8x4 blocks the splat's
// conservative alpha box overlaps (warp w = bxi + 2 byi owns the block whose
// pixel centres span [8 bxi + 0.5, 8 bxi + 7.5] x [4 byi + 0.5, 4 byi + 3.5]).
__device__ __forceinline__ BlendRec make_blend_rec(const Gauss64* __restrict__ g64,
                                                   const Gauss32* __restrict__ g32, uint32_t gi,
                                                   int tx0, int ty0) {
    const double2 m = *reinterpret_cast<const double2*>(&g32[gi].mx);
    const float4 q0 = *reinterpret_cast<const float4*>(&g32[gi].ha);
    const float4 col = *reinterpret_cast<const float4*>(&g32[gi].op);
    const float2 h = *reinterpret_cast<const float2*>(&g32[gi].hx);
    const float mtx = float(m.x - double(tx0));
    const float mty = float(m.y - double(ty0));
    uint32_t mask = 0;
    if (h.x >= 0.0f) {
        const uint32_t xm = (mtx - h.x <= 7.5f && mtx + h.x >= 0.5f ? 1u : 0u) |
                            (mtx - h.x <= 15.5f && mtx + h.x >= 8.5f ? 2u : 0u);
#pragma unroll
        for (int v = 0; v < 4; ++v)
            if (mty - h.y <= 4.0f * v + 3.5f && mty + h.y >= 4.0f * v + 0.5f) mask |= xm << (2 * v);
    }
    BlendRec r;
    r.geo = make_float4(mtx, mty, q0.x, q0.z);
    r.ct = make_float4(q0.y, q0.w, col.x, col.y);
    r.gbm = make_float4(col.z, col.w, __uint_as_float(mask), __uint_as_float(gi));
    return r;
}

// The record for the key placed at global pair position p of `tile`.
__device__ __forceinline__ void emit_rec(const RecOut& ro, uint32_t p, unsigned long long key,
                                         uint32_t tile, int tiles_x) {
    if (!ro.rec) return;
    ro.rec[p] = make_blend_rec(ro.g64, ro.g32, uint32_t(key), int(tile % uint32_t(tiles_x)) * kTile,
                               int(tile / uint32_t(tiles_x)) * kTile);
}
#endif

}  // namespace fgs
