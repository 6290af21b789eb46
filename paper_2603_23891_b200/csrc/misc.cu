// misc.cu -- small device utilities: tree packing at upload, run totals,
// tile-id range for the standalone sort.
#include "launch.h"

namespace fgs {

// SoA upload -> float4 quaternions (filter) + 64-byte splat records
// (preprocess gather).  soa = [mx|my|mz|sx|sy|sz], extra = [qw|qx|qy|qz|op|cr|cg|cb].
__global__ void k_pack_tree(const float* __restrict__ soa, uint64_t stride,
                            const float* __restrict__ ex, uint64_t n, float4* quat,
                            SplatRec* splat) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    SplatRec r;
    r.mx = soa[i];
    r.my = soa[stride + i];
    r.mz = soa[2 * stride + i];
    r.sx = soa[3 * stride + i];
    r.sy = soa[4 * stride + i];
    r.sz = soa[5 * stride + i];
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
    quat[i] = make_float4(r.qw, r.qx, r.qy, r.qz);
    splat[i] = r;
}

void launch_pack_tree(const float* soa, uint64_t stride, const float* extra, uint64_t n,
                      float4* quat, SplatRec* splat, cudaStream_t s) {
    if (n) k_pack_tree<<<unsigned((n + 255) / 256), 256, 0, s>>>(soa, stride, extra, n, quat, splat);
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

}  // namespace fgs
