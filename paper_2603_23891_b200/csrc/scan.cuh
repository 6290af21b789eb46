// scan.cuh -- single-pass chained scan (decoupled look-back) for ordered
// stream compaction.  Each CTA takes a ticket (so tiles are claimed in order
// and every predecessor is already resident: no deadlock), publishes its
// aggregate, then looks back warp-wide over up to 32 predecessors at a time
// until it meets an inclusive prefix.  Used by the filter's selected-list
// compaction (filter.cpp:147-148 "ordered") and by preprocess's gaussian
// compaction (rasterizer.cpp:54-71 keeps selected order).
#pragma once

#include <cstdint>

namespace fgs {

// status word: [63:62] flag (0 empty, 1 aggregate, 2 inclusive prefix), [61:0] value
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Called by ONE full warp of the CTA (lane 0 holds `aggregate`).  Returns the
// exclusive prefix for `tile` in all lanes.
__device__ __forceinline__ unsigned long long chained_scan_warp(unsigned long long* status,
                                                                unsigned int tile,
                                                                unsigned long long aggregate) {
    const unsigned lane = threadIdx.x & 31;
    aggregate = __shfl_sync(0xffffffffu, aggregate, 0);
    if (tile == 0) {
        if (lane == 0) st_release_u64(&status[0], kFlagPre | aggregate);
        return 0;
    }
    if (lane == 0) st_release_u64(&status[tile], kFlagAgg | aggregate);
    unsigned long long exclusive = 0;
    int base = int(tile) - 1;  // predecessor examined by lane 0
    while (true) {
        const int t = base - int(lane);
        unsigned long long w = kFlagPre;  // virtual predecessors (< 0) are empty prefixes
        if (t >= 0) {
            do {
                w = ld_volatile_u64(&status[t]);
            } while ((w >> 62) == 0);
        }
        const unsigned pre_mask = __ballot_sync(0xffffffffu, (w >> 62) == 2);
        // lanes 0..k where k = first lane holding an inclusive prefix
        const int k = pre_mask ? __ffs(pre_mask) - 1 : 31;
        unsigned long long v = (int(lane) <= k) ? (w & kValMask) : 0ull;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        exclusive += __shfl_sync(0xffffffffu, v, 0);
        if (pre_mask) break;
        base -= 32;
    }
    if (lane == 0) st_release_u64(&status[tile], kFlagPre | (exclusive + aggregate));
    return exclusive;
}

// Dynamic, ordered tile ticket (thread 0), broadcast through shared memory.
__device__ __forceinline__ unsigned int take_ticket(unsigned int* counter, unsigned int* smem) {
    __syncthreads();
    if (threadIdx.x == 0) *smem = atomicAdd(counter, 1u);
    __syncthreads();
    return *smem;
}

}  // namespace fgs
