// sort.cu -- per-tile segment sort: the remaining digits of the (tile, depth)
// radix sort.
//
// The reference sorts all pairs with an LSD radix on
// key = tile << 32 | bits(depth) and relies on stability to keep ties in
// gaussian order (rasterizer.cpp:100-135).  Here the tile digit was already
// resolved by counting (preprocess.cu scatters every key into its tile's
// bucket), so what is left is ordering each bucket by depth_bits << 32 |
// gaussian -- a total order with no ties, identical to the stable order.
// Buckets are sorted in shared memory (the whole bucket is resident: mean
// 290, p99 810 pairs per tile on the 10M tree), so the only HBM/L2 traffic
// of the sort is one read and one write of each 8-byte key.
//
// The in-shared-memory network is the direction-free ("flip") bitonic
// sorter: every comparator is oriented low->high, so a non-power-of-two
// bucket is padded virtually with +inf (a comparator whose high index is
// past the end is skipped and the padding never moves).
#include "blend_rec.cuh"
#include "launch.h"
#include "pdl.cuh"

namespace fgs {

// Where a sort places a bucket's keys for good: the blend records of those
// positions are written alongside (RecOut::rec, the TMA-staged blend); null
// for sorts into shared memory (runs, whose final positions come later).
struct RecSite {
    RecOut ro;
    uint32_t pbase;  // global pair index of the bucket's first key
    uint32_t tile;
    int tiles_x;
    __device__ __forceinline__ void put(uint32_t i, unsigned long long key) const {
        emit_rec(ro, pbase + i, key, tile, tiles_x);
    }
};

template <typename Index, typename Sync>
__device__ __forceinline__ void flip_bitonic(unsigned long long* a, Index n, Index tid,
                                             Index nthreads, Sync sync) {
    Index p = 1;
    while (p < n) p <<= 1;
    const Index half = p >> 1;
    for (Index k = 2; k <= p; k <<= 1) {
        const Index hk = k >> 1;
        for (Index c = tid; c < half; c += nthreads) {
            const Index blk = c / hk, off = c - blk * hk;
            const Index lo = blk * k + off, hi = blk * k + k - 1 - off;
            if (hi < n) {
                const unsigned long long x = a[lo], y = a[hi];
                if (y < x) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
        }
        sync();
        for (Index j = k >> 2; j >= 1; j >>= 1) {
            for (Index c = tid; c < half; c += nthreads) {
                const Index blk = c / j, off = c - blk * j;
                const Index lo = blk * 2 * j + off, hi = lo + j;
                if (hi < n) {
                    const unsigned long long x = a[lo], y = a[hi];
                    if (y < x) {
                        a[lo] = y;
                        a[hi] = x;
                    }
                }
            }
            sync();
        }
    }
}

constexpr int kSmallSortThreads = 256;
constexpr uint32_t kRun = 1024;  // run length of the run-sort + rank-merge path

// Barriers over the threads that sort one bucket (or one run): the whole
// 256-thread CTA of k_tile_sort, or one 256-thread group of k_tile_sort_big
// (named barrier per group).
struct CtaBar {
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ bool sync_or(bool p) const { return __syncthreads_or(p); }
};
struct GroupBar {
    unsigned id;
    __device__ __forceinline__ void sync() const {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kSmallSortThreads) : "memory");
    }
    __device__ __forceinline__ bool sync_or(bool p) const {
        unsigned r;
        asm volatile(
            "{ .reg .pred q, o;\n\t"
            "setp.ne.u32 q, %1, 0;\n\t"
            "bar.red.or.pred o, %2, %3, q;\n\t"
            "selp.u32 %0, 1, 0, o; }"
            : "=r"(r)
            : "r"(unsigned(p)), "r"(id), "r"(kSmallSortThreads)
            : "memory");
        return r != 0;
    }
};

__device__ __forceinline__ unsigned long long shfl_xor_u64(unsigned long long v, int m) {
    const unsigned lo = __shfl_xor_sync(0xffffffffu, unsigned(v), m);
    const unsigned hi = __shfl_xor_sync(0xffffffffu, unsigned(v >> 32), m);
    return (unsigned long long)hi << 32 | lo;
}

// Compare-exchange step of element i (partner i ^ j) in a bitonic network of
// stage k: keep the smaller value iff (i is the lower of the pair) == (the
// block of size k is ascending).
__device__ __forceinline__ unsigned long long bitonic_pick(unsigned long long mine,
                                                           unsigned long long other, uint32_t i,
                                                           uint32_t j, uint32_t k) {
    const bool keep_min = ((i & j) == 0) == ((i & k) == 0);
    return (other < mine) == keep_min ? other : mine;
}

// Buckets of up to 256*R keys: bitonic network over P = 2^ceil(log2 n) >= 32
// slots, padded with +inf.  Slot i = r * 256 + tid lives in register r of
// thread tid, so partners at distance j < 32 are exchanged with warp shuffles,
// 32 <= j < 256 through (double-buffered) shared memory with one named barrier
// (xbar) over the threads in play, j >= 256 inside the thread.  Only warps
// owning slots < P take part: a 40-key bucket is one warp and never waits.
// P is a compile-time power of two (32..1024): every stage below unrolls with
// constant distances, so the network is straight-line code.  keys -> out
// (global or shared); tid is the thread's index among the 256 sorting threads.
template <int LOGP>
__device__ __forceinline__ void register_bitonic(const unsigned long long* keys, uint32_t n,
                                                 unsigned long long* out,
                                                 unsigned long long* s_x, uint32_t tid,
                                                 unsigned xbar, const RecSite* site = nullptr) {
    constexpr uint32_t P = 1u << LOGP;
    constexpr int R = P > uint32_t(kSmallSortThreads) ? int(P / kSmallSortThreads) : 1;
    constexpr uint32_t lanes = P < uint32_t(kSmallSortThreads) ? P : uint32_t(kSmallSortThreads);
    if (tid >= lanes) return;  // whole warps (lanes is a multiple of 32)
    unsigned long long v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = uint32_t(r) * kSmallSortThreads + tid;
        v[r] = i < n ? keys[i] : ~0ull;
    }
    int parity = 0;
#pragma unroll
    for (uint32_t k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            if (j >= uint32_t(kSmallSortThreads)) {
                // partners in registers r and r ^ (j / 256); indices kept static
                auto cas = [&](unsigned long long& a, unsigned long long& b, int r) {
                    const uint32_t i = uint32_t(r) * kSmallSortThreads + tid;
                    const bool up = (i & k) == 0;
                    const bool sw = up ? (b < a) : (a < b);
                    const unsigned long long lo = sw ? b : a, hi = sw ? a : b;
                    a = lo;
                    b = hi;
                };
                if constexpr (R == 2) {
                    cas(v[0], v[1], 0);
                } else if constexpr (R == 4) {
                    if (j == uint32_t(kSmallSortThreads)) {
                        cas(v[0], v[1], 0);
                        cas(v[2], v[3], 2);
                    } else {
                        cas(v[0], v[2], 0);
                        cas(v[1], v[3], 1);
                    }
                }
            } else if (j >= 32) {
                unsigned long long* buf = s_x + (parity ? R * kSmallSortThreads : 0);
                parity ^= 1;
#pragma unroll
                for (int r = 0; r < R; ++r) buf[r * kSmallSortThreads + tid] = v[r];
                asm volatile("bar.sync %0, %1;" ::"r"(xbar), "r"(lanes) : "memory");
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t i = uint32_t(r) * kSmallSortThreads + tid;
                    v[r] = bitonic_pick(v[r], buf[r * kSmallSortThreads + (tid ^ j)], i, j, k);
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t i = uint32_t(r) * kSmallSortThreads + tid;
                    v[r] = bitonic_pick(v[r], shfl_xor_u64(v[r], int(j)), i, j, k);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = uint32_t(r) * kSmallSortThreads + tid;
        if (i < n) {
            out[i] = v[r];
            if (site) site->put(i, v[r]);
        }
    }
}

// Odd-even transposition over s_out[0, n) until no adjacent pair is out of
// order: moves keys only inside runs of equal depth (the input is sorted by
// depth), which puts ties into slot order -- the reference's stable order.
template <class Bar>
__device__ __forceinline__ void oddeven_fix(unsigned long long* s_out, uint32_t n, uint32_t tid,
                                            Bar bar) {
    while (true) {
        bool swapped = false;
#pragma unroll
        for (int ph = 0; ph < 2; ++ph) {
            for (uint32_t p = tid; 2 * p + ph + 1 < n; p += kSmallSortThreads) {
                const uint32_t a = 2 * p + ph;
                const unsigned long long x = s_out[a], y = s_out[a + 1];
                if (y < x) {
                    s_out[a] = y;
                    s_out[a + 1] = x;
                    swapped = true;
                }
            }
            bar.sync();
        }
        if (!bar.sync_or(swapped)) break;
    }
}

// 32-bit variant of the register network for buckets whose depth bits span
// less than 2^20 (a tile's splats sit in a narrow depth band): key32 =
// (depth_bits - min) << 12 | position in the bucket.  Half the shuffles, one
// compare and one select per exchange.  Equal depth bits then come out in
// bucket order, not slot order, so the gathered 64-bit keys get odd-even
// transposition passes until stable -- adjacent swaps only ever happen inside
// runs of equal depth, which are short.  Returns false (nothing written) when
// the bucket's depth range is too wide; the caller then runs the 64-bit
// network.  All 256 threads of the sorting group must call it.
// Shared memory: s_orig (P keys), s_x (2P words), s_red (16 words); the sorted
// keys land in s_out (shared) and, when dst is set, are copied there.
template <int LOGP, class Bar>
__device__ __forceinline__ bool register_bitonic32(const unsigned long long* keys, uint32_t n,
                                                   unsigned long long* s_orig, uint32_t* s_x,
                                                   uint32_t* s_red, unsigned long long* s_out,
                                                   unsigned long long* dst, uint32_t tid,
                                                   unsigned xbar, Bar bar,
                                                   const RecSite* site = nullptr) {
    constexpr uint32_t P = 1u << LOGP;
    constexpr int R = P > uint32_t(kSmallSortThreads) ? int(P / kSmallSortThreads) : 1;
    constexpr uint32_t lanes = P < uint32_t(kSmallSortThreads) ? P : uint32_t(kSmallSortThreads);
    static_assert(P <= 1024, "positions take 12 bits, the staging 8 KB");
    const unsigned lane = tid & 31, warp = tid >> 5;
    unsigned long long v[R];
    uint32_t dmin = 0xFFFFFFFFu, dmax = 0u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = uint32_t(r) * kSmallSortThreads + tid;
        v[r] = (tid < lanes && i < n) ? keys[i] : ~0ull;
        if (tid < lanes && i < n) {
            s_orig[i] = v[r];
            const uint32_t d = uint32_t(v[r] >> 32);
            dmin = min(dmin, d);
            dmax = max(dmax, d);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        dmin = min(dmin, __shfl_xor_sync(0xffffffffu, dmin, off));
        dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
    }
    if (lane == 0) {
        s_red[warp] = dmin;
        s_red[kSmallSortThreads / 32 + warp] = dmax;
    }
    bar.sync();
#pragma unroll
    for (int w = 0; w < kSmallSortThreads / 32; ++w) {
        dmin = min(dmin, s_red[w]);
        dmax = max(dmax, s_red[kSmallSortThreads / 32 + w]);
    }
    if (dmax - dmin >= (1u << 20)) return false;  // uniform across the group
    uint32_t k32[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = uint32_t(r) * kSmallSortThreads + tid;
        k32[r] = i < n ? ((uint32_t(v[r] >> 32) - dmin) << 12 | i) : 0xFFFFFFFFu;
    }
    if (tid < lanes) {
        int parity = 0;
#pragma unroll
        for (uint32_t k = 2; k <= P; k <<= 1) {
#pragma unroll
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                if (j >= uint32_t(kSmallSortThreads)) {
                    auto cas = [&](uint32_t& a, uint32_t& c, int r) {
                        const uint32_t i = uint32_t(r) * kSmallSortThreads + tid;
                        const bool up = (i & k) == 0;
                        const uint32_t lo = min(a, c), hi = max(a, c);
                        a = up ? lo : hi;
                        c = up ? hi : lo;
                    };
                    if constexpr (R == 2) {
                        cas(k32[0], k32[1], 0);
                    } else if constexpr (R == 4) {
                        if (j == uint32_t(kSmallSortThreads)) {
                            cas(k32[0], k32[1], 0);
                            cas(k32[2], k32[3], 2);
                        } else {
                            cas(k32[0], k32[2], 0);
                            cas(k32[1], k32[3], 1);
                        }
                    }
                } else if (j >= 32) {
                    uint32_t* buf = s_x + (parity ? R * kSmallSortThreads : 0);
                    parity ^= 1;
#pragma unroll
                    for (int r = 0; r < R; ++r) buf[r * kSmallSortThreads + tid] = k32[r];
                    asm volatile("bar.sync %0, %1;" ::"r"(xbar), "r"(lanes) : "memory");
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const uint32_t i = uint32_t(r) * kSmallSortThreads + tid;
                        const uint32_t o = buf[r * kSmallSortThreads + (tid ^ j)];
                        const bool keep_min = ((i & j) == 0) == ((i & k) == 0);
                        k32[r] = keep_min ? min(o, k32[r]) : max(o, k32[r]);
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const uint32_t i = uint32_t(r) * kSmallSortThreads + tid;
                        const uint32_t o = __shfl_xor_sync(0xffffffffu, k32[r], int(j));
                        const bool keep_min = ((i & j) == 0) == ((i & k) == 0);
                        k32[r] = keep_min ? min(o, k32[r]) : max(o, k32[r]);
                    }
                }
            }
        }
    }
    bar.sync();  // s_orig complete everywhere
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = uint32_t(r) * kSmallSortThreads + tid;
        if (tid < lanes && i < n) s_out[i] = s_orig[k32[r] & 0xFFFu];
    }
    bar.sync();
    oddeven_fix(s_out, n, tid, bar);  // runs of equal depth into slot order
    if (dst)
        for (uint32_t i = tid; i < n; i += kSmallSortThreads) {
            dst[i] = s_out[i];
            if (site) site->put(i, s_out[i]);
        }
    return true;
}

// LSD radix sort of one bucket (n <= 256 R keys) by depth: the remaining
// digits of the reference's (tile, depth) radix sort (rasterizer.cpp:100-135)
// once the tile digit has been resolved by counting (k_emit_keys).  Digits are
// taken from depth_bits - min over the bucket, only as many as its depth range
// spans (a tile's splats sit in a narrow band: typically 2-3 passes), at most
// 8 bits each; every pass is stable, so equal depths keep their bucket order
// and oddeven_fix then puts them into slot order.
// Warp w holds the 32 R consecutive positions [32 R w, 32 R (w + 1)), lane l
// position 32 R w + 32 r + l of round r.  A key's rank: the count of its digit
// in the warp's earlier rounds (one shared counter per (warp, digit), bumped
// by the lowest lane of each __match_any_sync group) + its rank in the group;
// one CTA-wide exclusive scan over (digit, warp) turns the counters into
// destinations.  Shared memory (s, 32 KB): two key buffers of 1024 and two
// counter arrays [8][256] (alternating passes, the idle one zeroed during the
// scan).  The sorted bucket goes to dst (global) and, for the TMA blend, its
// records through `site`.
template <int R>
__device__ __forceinline__ void radix_bucket(const unsigned long long* __restrict__ keys,
                                             uint32_t n, unsigned long long* dst,
                                             unsigned long long* s, uint32_t* s_red, uint32_t tid,
                                             const RecSite* site) {
    static_assert(R >= 1 && 32 * R * (kSmallSortThreads / 32) <= 1024, "1024 keys at most");
    constexpr uint32_t kSeg = 32u * R;
    constexpr int kWarps = kSmallSortThreads / 32;
    const uint32_t lane = tid & 31, warp = tid >> 5;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(s + 2048);  // [2][kWarps][256]
    unsigned long long v[R];
    uint32_t dmin = 0xFFFFFFFFu, dmax = 0u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t p = kSeg * warp + 32u * r + lane;
        v[r] = p < n ? keys[p] : ~0ull;
        if (p < n) {
            const uint32_t d = uint32_t(v[r] >> 32);
            dmin = min(dmin, d);
            dmax = max(dmax, d);
        }
    }
    for (uint32_t j = tid; j < 2u * kWarps * 256u; j += kSmallSortThreads) cnt[j] = 0u;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        dmin = min(dmin, __shfl_xor_sync(0xffffffffu, dmin, off));
        dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
    }
    if (lane == 0) {
        s_red[warp] = dmin;
        s_red[kWarps + warp] = dmax;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        dmin = min(dmin, s_red[w]);
        dmax = max(dmax, s_red[kWarps + w]);
    }
    const uint32_t range = dmax - dmin;
    const int nbits = range ? 32 - __clz(range) : 0;
    const int passes = (nbits + 7) >> 3;
    const int width = passes ? (nbits + passes - 1) / passes : 0;
    const uint32_t mask = (1u << width) - 1u, bins = 1u << width;
    unsigned long long* out = s;
    __syncthreads();  // s_red is reused by the scans
    for (int ps = 0; ps < passes; ++ps) {
        uint32_t* c = cnt + (ps & 1) * (kWarps * 256);
        const int shift = ps * width;
        uint32_t dig[R], rank[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t p = kSeg * warp + 32u * r + lane;
            const bool ok = p < n;
            // lanes past n get a private digit: never in anyone's group
            const uint32_t d = ok ? ((uint32_t(v[r] >> 32) - dmin) >> shift) & mask : 256u + lane;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const uint32_t below = __popc(peers & ((1u << lane) - 1u));
            const uint32_t base = ok ? c[warp * 256u + d] : 0u;
            __syncwarp();
            if (ok && below == 0) c[warp * 256u + d] = base + __popc(peers);
            __syncwarp();
            dig[r] = d;
            rank[r] = base + below;
        }
        __syncthreads();
        // exclusive scan over (digit, warp); thread t owns digit t
        uint32_t row[kWarps], tot = 0u;
        if (tid < bins) {
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                row[w] = c[w * 256u + tid];
                tot += row[w];
            }
        }
        uint32_t incl = tot;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= uint32_t(off)) incl += t;
        }
        if (lane == 31) s_red[warp] = incl;
        __syncthreads();
        uint32_t off = incl - tot;
        for (uint32_t w = 0; w < warp; ++w) off += s_red[w];
        if (tid < bins) {
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                c[w * 256u + tid] = off;
                off += row[w];
            }
        }
        {  // the other counter array (last read by the previous pass) for the next pass
            uint32_t* c2 = cnt + ((ps + 1) & 1) * (kWarps * 256);
#pragma unroll
            for (int w = 0; w < kWarps; ++w) c2[w * 256u + tid] = 0u;
        }
        __syncthreads();
        out = s + (ps & 1) * 1024;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t p = kSeg * warp + 32u * r + lane;
            if (p < n) out[c[warp * 256u + dig[r]] + rank[r]] = v[r];
        }
        __syncthreads();
        if (ps + 1 < passes) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t p = kSeg * warp + 32u * r + lane;
                v[r] = p < n ? out[p] : ~0ull;
            }
        }
    }
    if (passes == 0) {  // one depth: bucket order, to be put into slot order
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t p = kSeg * warp + 32u * r + lane;
            if (p < n) out[p] = v[r];
        }
        __syncthreads();
    }
    oddeven_fix(out, n, tid, CtaBar{});
    for (uint32_t i = tid; i < n; i += kSmallSortThreads) {
        dst[i] = out[i];
        if (site) site->put(i, out[i]);
    }
}

// One run of up to kRun keys (global) sorted into shared memory by 256
// threads: the 32-bit network when the run's depth band allows, else the
// 64-bit one.  stage: kRun keys of staging (s_orig, then the exchange words;
// the 64-bit network's double buffer reuses all of it).
template <class Bar>
__device__ __forceinline__ void sort_run(const unsigned long long* keys, uint32_t n,
                                         unsigned long long* s_run, unsigned long long* stage,
                                         uint32_t* s_red, uint32_t tid, unsigned xbar, Bar bar) {
    if (register_bitonic32<10>(keys, n, stage, reinterpret_cast<uint32_t*>(stage + kRun), s_red,
                               s_run, nullptr, tid, xbar, bar))
        return;
    bar.sync();  // staging reused by the 64-bit network
    register_bitonic<10>(keys, n, s_run, stage, tid, xbar);
}

// Sorted runs of kRun keys in shared memory -> the sorted bucket in dst.  Keys
// are unique (the low word is the emission slot), so a key's final position is
// its index in its run plus, for every other run, the number of keys below it
// (a fixed-depth binary search); each key is stored once, straight to HBM.
__device__ __forceinline__ void rank_merge(const unsigned long long* runs, uint32_t n,
                                           unsigned long long* dst, uint32_t tid, uint32_t nthr,
                                           const RecSite& site) {
    const uint32_t n_runs = (n + kRun - 1) / kRun;
    for (uint32_t i = tid; i < n; i += nthr) {
        const unsigned long long x = runs[i];
        const uint32_t r = i / kRun;
        uint32_t rank = i - r * kRun;
        for (uint32_t q = 0; q < n_runs; ++q) {
            if (q == r) continue;
            const unsigned long long* run = runs + q * kRun;
            const uint32_t len = min(kRun, n - q * kRun);
            uint32_t pos = 0;
#pragma unroll
            for (uint32_t step = kRun; step > 0; step >>= 1)
                if (pos + step <= len && run[pos + step - 1] < x) pos += step;
            rank += pos;
        }
        dst[rank] = x;
        site.put(rank, x);
    }
}

// CTAs per SM the register budget is cut for.  The per-bucket sort is latency-bound,
// so occupancy wins at 1080p -- 4 / 5 / 6 CTAs (56 / 48 / 40 registers; 6 spills 16
// bytes, and the 33.8 KB of shared memory caps it there): tile sort 49.4 / 45.6 / 44.1 us
// per cfg-3 frame -- but at 4K, where many buckets take the two-run path, 6 loses 9 % of
// cfg 4's frame rate to 5 (527 vs 576 frames/s).  Both are built, chosen per frame size.
constexpr int kSortCtasSmall = 6, kSortCtasBig = 5;
constexpr int kSortBigFrameTiles = 12288;
template <int kCtas>
__global__ void __launch_bounds__(kSmallSortThreads, kCtas) k_tile_sort(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ order,
    unsigned long long* keys, const RecOut ro, const int tiles_x) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    static_assert(kSmallSortCap == 2 * int(kRun), "two runs + their staging fill s");
    __shared__ unsigned long long s[2 * kSmallSortCap];
    __shared__ uint32_t s_red[2 * kSmallSortThreads / 32];
    const uint32_t tile = order[blockIdx.x];  // heaviest buckets first
    const uint32_t b = offsets[tile], e = offsets[tile + 1];
    const uint32_t n = e - b;
    const uint32_t tid = threadIdx.x;
    const RecSite site{ro, b, tile, tiles_x};
    if (n == 1 && tid == 0) site.put(0, keys[b]);
    if (n < 2 || n > uint32_t(kSmallSortCap)) return;  // big buckets: k_tile_sort_big
    const RecSite* sp = ro.rec ? &site : nullptr;
#ifndef SORT32
#define SORT32 1
#endif
    if (n > kRun) {  // two runs, then the rank merge
        for (uint32_t r = 0; r * kRun < n; ++r) {
            sort_run(keys + b + r * kRun, min(kRun, n - r * kRun), s + r * kRun,
                     s + kSmallSortCap, s_red, tid, 1, CtaBar{});
            __syncthreads();
        }
        rank_merge(s, n, keys + b, tid, kSmallSortThreads, site);
        return;
    }
#ifndef SORT_RADIX
#define SORT_RADIX 0  // per-tile LSD radix (measured slower: DESIGN.md 3)
#endif
#if SORT_RADIX
    if (n > 64u) {
        if (n <= 256u) radix_bucket<1>(keys + b, n, keys + b, s, s_red, tid, sp);
        else if (n <= 512u) radix_bucket<2>(keys + b, n, keys + b, s, s_red, tid, sp);
        else radix_bucket<4>(keys + b, n, keys + b, s, s_red, tid, sp);
        return;
    }
#endif
#if SORT32
    {
        bool done;
        uint32_t* sx32 = reinterpret_cast<uint32_t*>(s + kRun);
        unsigned long long* so = s + 2 * kRun;
        if (n <= 32u) done = register_bitonic32<5>(keys + b, n, s, sx32, s_red, so, keys + b, tid, 1, CtaBar{}, sp);
        else if (n <= 64u) done = register_bitonic32<6>(keys + b, n, s, sx32, s_red, so, keys + b, tid, 1, CtaBar{}, sp);
        else if (n <= 128u) done = register_bitonic32<7>(keys + b, n, s, sx32, s_red, so, keys + b, tid, 1, CtaBar{}, sp);
        else if (n <= 256u) done = register_bitonic32<8>(keys + b, n, s, sx32, s_red, so, keys + b, tid, 1, CtaBar{}, sp);
        else if (n <= 512u) done = register_bitonic32<9>(keys + b, n, s, sx32, s_red, so, keys + b, tid, 1, CtaBar{}, sp);
        else done = register_bitonic32<10>(keys + b, n, s, sx32, s_red, so, keys + b, tid, 1, CtaBar{}, sp);
        if (done) return;
        __syncthreads();  // staging in s is reused by the 64-bit network
    }
#endif
    if (n <= 32u) register_bitonic<5>(keys + b, n, keys + b, s, tid, 1, sp);
    else if (n <= 64u) register_bitonic<6>(keys + b, n, keys + b, s, tid, 1, sp);
    else if (n <= 128u) register_bitonic<7>(keys + b, n, keys + b, s, tid, 1, sp);
    else if (n <= 256u) register_bitonic<8>(keys + b, n, keys + b, s, tid, 1, sp);
    else if (n <= 512u) register_bitonic<9>(keys + b, n, keys + b, s, tid, 1, sp);
    else register_bitonic<10>(keys + b, n, keys + b, s, tid, 1, sp);
}

constexpr int kBigGroups = 4;
constexpr int kBigSortThreads = kBigGroups * kSmallSortThreads;
constexpr int kBigSortSmem = (kBigSortCap + kBigGroups * 2 * int(kRun)) * 8;

// Buckets above kSmallSortCap: persistent CTAs (one per SM) take buckets from
// a queue; the bucket's runs of kRun keys are sorted by four 256-thread groups
// (named barriers 1-4 for the exchanges, 5-8 for the group) into shared
// memory, then all 1024 threads rank-merge them into place.  Beyond
// kBigSortCap the flip bitonic runs in place in global memory (L2-resident;
// only pathological tiles get there).
__global__ void __launch_bounds__(kBigSortThreads) k_tile_sort_big(const uint32_t* __restrict__ offsets,
                                                                   unsigned long long* keys,
                                                                   const uint32_t* big_list,
                                                                   FrameCounters* cnt,
                                                                   const RecOut ro,
                                                                   const int tiles_x) {
    pdl_wait();  // the previous kernel of the frame is complete and visible
    pdl_trigger();
    extern __shared__ unsigned long long s_big[];
    __shared__ uint32_t s_red[kBigGroups][2 * kSmallSortThreads / 32];
    __shared__ unsigned s_item;
    const unsigned n_big = cnt->big_tiles;
    const uint32_t g = threadIdx.x / kSmallSortThreads, gt = threadIdx.x % kSmallSortThreads;
    unsigned long long* stage = s_big + kBigSortCap + g * 2 * kRun;
    const GroupBar gbar{5u + g};
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) s_item = atomicAdd(&cnt->big_cursor, 1u);
        __syncthreads();
        const unsigned item = s_item;
        if (item >= n_big) break;
        const uint32_t tile = big_list[item];
        const uint32_t b = offsets[tile], e = offsets[tile + 1];
        const uint32_t n = e - b;
        if (n <= uint32_t(kBigSortCap)) {
            for (uint32_t r = g; r * kRun < n; r += kBigGroups) {
                sort_run(keys + b + r * kRun, min(kRun, n - r * kRun), s_big + r * kRun, stage,
                         s_red[g], gt, 1u + g, gbar);
                gbar.sync();  // staging reuse by the group's next run
            }
            __syncthreads();
            rank_merge(s_big, n, keys + b, threadIdx.x, kBigSortThreads, RecSite{ro, b, tile, tiles_x});
        } else {
            flip_bitonic<uint32_t>(keys + b, n, threadIdx.x, kBigSortThreads, [] __device__() {
                __threadfence_block();
                __syncthreads();
            });
            if (ro.rec) {
                const RecSite site{ro, b, tile, tiles_x};
                for (uint32_t i = threadIdx.x; i < n; i += kBigSortThreads) site.put(i, keys[b + i]);
            }
        }
    }
}

void launch_tile_sort(const uint32_t* offsets, const uint32_t* order, int n_tiles,
                      unsigned long long* keys, cudaStream_t s, RecOut ro, int tiles_x) {
    if (n_tiles <= 0) return;
    if (n_tiles > kSortBigFrameTiles)
        launch_pdl(k_tile_sort<kSortCtasBig>, n_tiles, kSmallSortThreads, 0, s, offsets, order,
                   keys, ro, tiles_x);
    else
        launch_pdl(k_tile_sort<kSortCtasSmall>, n_tiles, kSmallSortThreads, 0, s, offsets, order,
                   keys, ro, tiles_x);
}

void launch_tile_sort_big(const uint32_t* offsets, unsigned long long* keys,
                          const uint32_t* big_list, FrameCounters* cnt, int grid,
                          cudaStream_t s, RecOut ro, int tiles_x) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_tile_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kBigSortSmem);
        attr = true;
    }
    launch_pdl(k_tile_sort_big, grid, kBigSortThreads, kBigSortSmem, s, offsets, keys, big_list,
               cnt, ro, tiles_x);
}

// ----------------------------------------------------------------------------
// Stage-entry helpers for the standalone sort_pairs / alpha_blend.

__global__ void k_bucket_triples(const uint32_t* t, uint64_t n, uint32_t* count) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) atomicAdd(count + t[i * 3], 1u);
}

void launch_bucket_triples(const uint32_t* triples, uint64_t n, uint32_t* tile_count,
                           cudaStream_t s) {
    if (n) k_bucket_triples<<<unsigned((n + 255) / 256), 256, 0, s>>>(triples, n, tile_count);
}

// key = depth bits << 32 | input position: stable order == reference order.
__global__ void k_scatter_triples(const uint32_t* t, uint64_t n, uint32_t* cursor,
                                  unsigned long long* keys) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t pos = atomicAdd(cursor + t[i * 3], 1u);
    keys[pos] = (unsigned long long)t[i * 3 + 1] << 32 | i;
}

void launch_scatter_triples(const uint32_t* triples, uint64_t n, uint32_t* cursor,
                            unsigned long long* keys, cudaStream_t s) {
    if (n) k_scatter_triples<<<unsigned((n + 255) / 256), 256, 0, s>>>(triples, n, cursor, keys);
}

__global__ void k_gather_triples(const uint32_t* offsets, const unsigned long long* keys,
                                 const uint32_t* in, uint32_t* out) {
    const uint32_t tile = blockIdx.x;
    const uint32_t b = offsets[tile], e = offsets[tile + 1];
    for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        const uint32_t src = uint32_t(keys[i]);
        out[i * 3 + 0] = in[src * 3 + 0];
        out[i * 3 + 1] = in[src * 3 + 1];
        out[i * 3 + 2] = in[src * 3 + 2];
    }
}

void launch_gather_triples(const uint32_t* offsets, int n_tiles, const unsigned long long* keys,
                           const uint32_t* in_triples, uint32_t* out_triples, cudaStream_t s) {
    if (n_tiles > 0)
        k_gather_triples<<<n_tiles, 128, 0, s>>>(offsets, keys, in_triples, out_triples);
}

__global__ void k_triples_to_keys(const uint32_t* t, uint64_t n, unsigned long long* keys) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = (unsigned long long)t[i * 3 + 1] << 32 | t[i * 3 + 2];
}

void launch_triples_to_keys(const uint32_t* triples, uint64_t n, unsigned long long* keys,
                            cudaStream_t s) {
    if (n) k_triples_to_keys<<<unsigned((n + 255) / 256), 256, 0, s>>>(triples, n, keys);
}

__global__ void k_keys_to_triples(const uint32_t* offsets, const unsigned long long* keys,
                                  const uint32_t* g_of_slot, uint32_t* out) {
    const uint32_t tile = blockIdx.x;
    const uint32_t b = offsets[tile], e = offsets[tile + 1];
    for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        const unsigned long long k = keys[i];
        out[i * 3 + 0] = tile;
        out[i * 3 + 1] = uint32_t(k >> 32);
        out[i * 3 + 2] = g_of_slot ? g_of_slot[uint32_t(k)] : uint32_t(k);
    }
}

void launch_keys_to_triples(const uint32_t* offsets, int n_tiles, const unsigned long long* keys,
                            const uint32_t* g_of_slot, uint32_t* out_triples, cudaStream_t s) {
    if (n_tiles > 0)
        k_keys_to_triples<<<n_tiles, 128, 0, s>>>(offsets, keys, g_of_slot, out_triples);
}

}  // namespace fgs
