// Micro-benchmark: k_tile_offsets in isolation (CUDA events, 200 reps), to find
// where a 1-CTA scan over 8160 tile counts spends its time.
#include <cstdio>
#include <vector>
#include "../../paper_2603_23891_b200/csrc/launch.h"

namespace fgs {
void launch_tile_offsets(const uint32_t*, int, uint32_t*, uint32_t*, uint32_t*, uint32_t*,
                         FrameCounters*, uint64_t, cudaStream_t, RunTotals*);
}
namespace fgs {
__device__ __forceinline__ int tile_class(uint32_t c, uint32_t mean) {
    // 0: >= 4x mean pairs, 1: >= 2x, 2: >= 1x, 3: lighter
    return c >= 4 * mean ? 0 : (c >= 2 * mean ? 1 : (c >= mean ? 2 : 3));
}

__global__ void __launch_bounds__(1024) k_tile_offsets_t(const uint32_t* __restrict__ gcount,
                                                       int n_tiles, uint32_t* offsets,
                                                       uint32_t* cursor, uint32_t* big_list,
                                                       uint32_t* order, FrameCounters* cnt,
                                                       uint64_t pair_cap, RunTotals* totals,
                                                       int staged, unsigned long long* ts) {
    auto stamp = [&](int i) { __syncthreads(); if (threadIdx.x == 0) { unsigned long long v; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v)); ts[i] = v; } };
    stamp(0);
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
    stamp(1);
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
    stamp(2);
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
        if (totals) {
            totals->frames += 1;
            totals->sum_selected += cnt->n_selected;
            totals->sum_pairs += ovf ? 0ull : total;
            if (ovf) totals->pad = 1;
        }
    }
    stamp(3);
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
    stamp(4);
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
    stamp(5);
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
    stamp(6);
    if (staged) {
        __syncthreads();
        for (int t = threadIdx.x; t < n_tiles; t += 1024) order[t] = ord[t];
    }
    stamp(7);
}

}
using namespace fgs;

__global__ void k_empty() {}

int main() {
    const int n = 8160;
    std::vector<uint32_t> h(n);
    for (int i = 0; i < n; ++i) h[i] = (i * 2654435761u) % 600;
    uint32_t *c, *o, *cur, *big, *ord;
    FrameCounters* cnt;
    RunTotals* tot;
    cudaMalloc(&c, n * 4); cudaMalloc(&o, (n + 1) * 4); cudaMalloc(&cur, (n + 1) * 4);
    cudaMalloc(&big, (n + 1) * 4); cudaMalloc(&ord, (n + 1) * 4);
    cudaMalloc(&cnt, sizeof(FrameCounters)); cudaMalloc(&tot, sizeof(RunTotals));
    cudaMemcpy(c, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemset(cnt, 0, sizeof(FrameCounters));
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int variant = 0; variant < 3; ++variant) {
        for (int w = 0; w < 20; ++w) launch_tile_offsets(c, n, o, cur, big, ord, cnt, ~0ull, s, tot);
        cudaEventRecord(e0, s);
        for (int r = 0; r < 200; ++r) {
            if (variant == 0) launch_tile_offsets(c, n, o, cur, big, ord, cnt, ~0ull, s, tot);
            if (variant == 1) k_empty<<<1, 1024, 0, s>>>();
            if (variant == 2) k_empty<<<1, 32, 0, s>>>();
        }
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("variant %d: %.2f us per launch\n", variant, ms * 1000 / 200);
    }
    unsigned long long* ts;
    cudaMalloc(&ts, 64 * 8);
    cudaFuncSetAttribute(k_tile_offsets_t, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    for (int r = 0; r < 5; ++r) k_tile_offsets_t<<<1, 1024, (2 * n + 1) * 4, s>>>(c, n, o, cur, big, ord, cnt, ~0ull, tot, 1, ts);
    cudaDeviceSynchronize();
    unsigned long long h_ts[8];
    cudaMemcpy(h_ts, ts, 64, cudaMemcpyDeviceToHost);
    for (int i = 1; i < 8; ++i) printf("phase %d: %.2f us\n", i, (h_ts[i] - h_ts[i - 1]) / 1000.0);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
