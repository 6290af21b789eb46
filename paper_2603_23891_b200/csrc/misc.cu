// misc.cu -- small device utilities: tree packing at upload, run totals,
// tile-id range for the standalone sort.
#include <algorithm>

#include "launch.h"
#include "pdl.cuh"
#include "mark.cuh"

namespace fgs {

// SoA upload -> the device layout (launch.h DevTree): geo records for every
// node, scale/quaternion records for the internal region, 64-byte splat
// records.  soa = [mx|my|mz|sx|sy|sz] (stride n), ex = [qw|qx|qy|qz|op|cr|cg|cb].
__global__ void k_pack_tree(const float* __restrict__ soa, const float* __restrict__ ex,
                            const uint8_t* __restrict__ leaf, uint64_t n, uint64_t leaf_begin,
                            float4* geo, float4* iscale, float4* iquat, SplatRec* splat) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    SplatRec r;
    r.mx = soa[i];
    r.my = soa[n + i];
    r.mz = soa[2 * n + i];
    r.sx = soa[3 * n + i];
    r.sy = soa[4 * n + i];
    r.sz = soa[5 * n + i];
    r.qw = ex[i];
    r.qx = ex[n + i];
    r.qy = ex[2 * n + i];
    r.qz = ex[3 * n + i];
    r.opacity = ex[4 * n + i];
    r.cr = ex[5 * n + i];
    r.cg = ex[6 * n + i];
    r.cb = ex[7 * n + i];
    r.pad0 = 0.f;
    r.pad1 = 0.f;
    splat[i] = r;
    // std::max(std::max(sx, sy), sz) of mark_core.hpp:33, exact in float (scales finite > 0)
    const float smax = fmaxf(fmaxf(r.sx, r.sy), r.sz);
    geo[i] = make_float4(r.mx, r.my, r.mz, smax);
    if (i < leaf_begin) {
        iscale[i] = make_float4(r.sx, r.sy, r.sz, leaf[i] ? 1.0f : 0.0f);
        iquat[i] = make_float4(r.qw, r.qx, r.qy, r.qz);
    }
}

void launch_pack_tree(const float* soa, const float* extra, const uint8_t* leaf, uint64_t n,
                      uint64_t leaf_begin, float4* geo, float4* iscale, float4* iquat,
                      SplatRec* splat, cudaStream_t s) {
    if (n)
        k_pack_tree<<<unsigned((n + 255) / 256), 256, 0, s>>>(soa, extra, leaf, n, leaf_begin, geo,
                                                              iscale, iquat, splat);
}

__global__ void k_update_totals(const FrameCounters* cnt, const uint32_t* offsets, int n_tiles,
                                RunTotals* t) {
    t->frames += 1;
    t->sum_selected += cnt->n_selected;
    t->sum_pairs += offsets[n_tiles];
    if (cnt->overflow) t->pad = 1;
}

void launch_update_totals(const FrameCounters* cnt, const uint32_t* offsets, int n_tiles,
                          RunTotals* totals, cudaStream_t s) {
    k_update_totals<<<1, 1, 0, s>>>(cnt, offsets, n_tiles, totals);
}

__global__ void k_max_tile(const uint32_t* t, uint64_t n, unsigned int* out) {
    unsigned m = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        m = max(m, t[i * 3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

void launch_max_tile(const uint32_t* triples, uint64_t n, unsigned int* out, cudaStream_t s) {
    if (n) k_max_tile<<<148, 256, 0, s>>>(triples, n, out);
}

// Per-frame clearing of the counters / scan state / tile counts by a kernel:
// a cudaMemsetAsync may be served by a copy engine and would then queue
// behind the previous frame's image copy (render_batch overlaps the two).
__global__ void k_zero_words(uint4* p, uint64_t n16) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
         i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = make_uint4(0u, 0u, 0u, 0u);
}

void launch_zero(void* p, uint64_t bytes, cudaStream_t s) {
    const uint64_t n16 = bytes / 16;  // callers pass 256-byte multiples
    if (n16 == 0) return;
    const unsigned grid = unsigned(std::min<uint64_t>((n16 + 255) / 256, 148 * 4));
    launch_pdl(k_zero_words, grid, 256, 0, s, reinterpret_cast<uint4*>(p), n16);
}

// Banded blend of a synchronous frame (GpuScene::enqueue_pipeline): the frame's
// heavy-first tile order stably partitioned by horizontal band of band_rows tile rows,
// so band b's tiles occupy [b band_rows tiles_x, ...) of `out` in heavy-first order;
// the bands' blend tickets are cleared.  One CTA: thread k owns a contiguous run of
// the order, counts it per band, one block scan per band, a stable scatter.
constexpr int kBandThreads = 1024;
__global__ void __launch_bounds__(kBandThreads) k_band_order(const uint32_t* __restrict__ order,
                                                             const int n_tiles, const int tiles_x,
                                                             const int band_rows,
                                                             const int n_bands,
                                                             uint32_t* __restrict__ out,
                                                             unsigned* tickets) {
    pdl_wait();
    pdl_trigger();
    __shared__ uint32_t s_warp[kMaxBands][32];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < unsigned(n_bands)) tickets[tid] = 0u;
    const int per = (n_tiles + kBandThreads - 1) / kBandThreads;
    const int t0 = min(n_tiles, int(tid) * per), t1 = min(n_tiles, t0 + per);
    uint32_t cnt[kMaxBands];
#pragma unroll
    for (int b = 0; b < kMaxBands; ++b) cnt[b] = 0u;
    for (int i = t0; i < t1; ++i) {
        const int b = int(order[i]) / tiles_x / band_rows;
#pragma unroll
        for (int k = 0; k < kMaxBands; ++k) cnt[k] += k == b ? 1u : 0u;
    }
    // exclusive prefix of each band's counts over the threads
    uint32_t pre[kMaxBands];
#pragma unroll
    for (int b = 0; b < kMaxBands; ++b) {
        uint32_t incl = cnt[b];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= unsigned(o)) incl += v;
        }
        if (lane == 31) s_warp[b][warp] = incl;
        pre[b] = incl - cnt[b];
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < kMaxBands; ++b)
        for (unsigned w = 0; w < warp; ++w) pre[b] += s_warp[b][w];
    for (int i = t0; i < t1; ++i) {
        const uint32_t t = order[i];
        const int b = int(t) / tiles_x / band_rows;
#pragma unroll
        for (int k = 0; k < kMaxBands; ++k)
            if (k == b) out[uint32_t(k * band_rows * tiles_x) + pre[k]++] = t;
    }
}

void launch_band_order(const uint32_t* order, int n_tiles, int tiles_x, int band_rows,
                       int n_bands, uint32_t* out, unsigned* tickets, cudaStream_t s) {
    if (n_tiles <= 0) return;
    launch_pdl(k_band_order, 1, kBandThreads, 0, s, order, n_tiles, tiles_x, band_rows, n_bands,
               out, tickets);
}

}  // namespace fgs
