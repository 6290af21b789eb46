// ingest.cu -- scene ingest on the device.
//
// The reference validates the whole tree on every render (rasterizer.cpp:170,
// require_valid -> validate_tree, scene.cpp:89-165) and loads LDGS v1 files by
// de-interleaving on the host (scene_io.cpp:90-116).  Here a tree is
// validated once, on the device, when a GpuScene is created (from host arrays
// or straight from an LDGS file streamed through pinned buffers), and the
// file's interleaved sections are de-interleaved by a kernel.
//
// Validation reproduces the per-node rules of scene.cpp:125-162 bit for bit
// (the quaternion norm in FP64 with the reference's association, -fmad=false)
// as a 9-bit rule mask per node; the host turns the first masks into the
// reference's messages (host_util.cpp validate_tree wording).
#include "launch.h"

namespace fgs {

// scene.cpp:118-120: has_child[parent[i]] = 1 for in-range parents.
__global__ void k_has_child(const uint32_t* __restrict__ parent, uint64_t n,
                            uint8_t* __restrict__ has_child) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t p = parent[i];
    if (p != kRootParent && p < n) has_child[p] = 1;
}

__device__ __forceinline__ bool finite_f(float v) { return isfinite(v); }

// scene.cpp:122-162 per node.  soa = 14 arrays of n floats in the order
// mean xyz, scale xyz, quat wxyz, opacity, colour rgb.  Bits (rule order):
// 0 finite (exclusive), 1 unit quaternion, 2 scale > 0, 3 opacity in (0,1],
// 4 colour in [0,1], 5 level-0 parent is ROOT, 6 parent index in range,
// 7 parent level == level - 1, 8 leaf iff childless.
__global__ void k_validate_nodes(const float* __restrict__ soa, const uint32_t* __restrict__ parent,
                                 const uint8_t* __restrict__ leaf,
                                 const uint8_t* __restrict__ has_child, uint64_t n,
                                 const uint64_t* __restrict__ level_begin, int n_levels,
                                 uint16_t* __restrict__ mask, unsigned long long* n_bad) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned m = 0;
    if (i < n) {
        float v[14];
#pragma unroll
        for (int k = 0; k < 14; ++k) v[k] = soa[uint64_t(k) * n + i];
        bool fin = true;
#pragma unroll
        for (int k = 0; k < 14; ++k) fin = fin && finite_f(v[k]);
        if (!fin) {
            m = 1u;
        } else {
            const double qw = v[6], qx = v[7], qy = v[8], qz = v[9];
            const double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
            if (fabs(qn - 1.0) > 1e-6) m |= 1u << 1;
            if (!(v[3] > 0 && v[4] > 0 && v[5] > 0)) m |= 1u << 2;
            if (!(v[10] > 0 && v[10] <= 1)) m |= 1u << 3;
            if (!(v[11] >= 0 && v[11] <= 1 && v[12] >= 0 && v[12] <= 1 && v[13] >= 0 &&
                  v[13] <= 1))
                m |= 1u << 4;
            // level of a node: last level whose begin <= index (offsets validated on host)
            auto level_of = [&](uint64_t x) {
                int lo = 0, hi = n_levels - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (level_begin[mid] <= x) lo = mid;
                    else hi = mid - 1;
                }
                return lo;
            };
            const int li = level_of(i);
            const uint32_t p = parent[i];
            if (li == 0) {
                if (p != kRootParent) m |= 1u << 5;
            } else if (p == kRootParent || p >= n) {
                m |= 1u << 6;
            } else if (level_of(p) + 1 != li) {
                m |= 1u << 7;
            }
            if ((leaf[i] != 0) == (has_child[i] != 0)) m |= 1u << 8;
        }
        mask[i] = uint16_t(m);
    }
    unsigned c = __popc(m);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(n_bad, (unsigned long long)c);
}

// scene_io.cpp:90-116 load_binary: the payload after the 20-byte header,
// sections back to back -- means (xyz per node), scales (xyz), quaternions
// (wxyz), opacity, colours (rgb), parents (u32), leaf flags (u8) -- into the
// 14 float SoA arrays + parent + leaf of the ingest staging.
__global__ void k_deinterleave(const uint8_t* __restrict__ payload, uint64_t n,
                               float* __restrict__ soa, uint32_t* __restrict__ parent,
                               uint8_t* __restrict__ leaf) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* means = reinterpret_cast<const float*>(payload);
    const float* scales = means + 3 * n;
    const float* quats = scales + 3 * n;
    const float* opac = quats + 4 * n;
    const float* cols = opac + n;
    const uint32_t* par = reinterpret_cast<const uint32_t*>(cols + 3 * n);
    const uint8_t* lf = reinterpret_cast<const uint8_t*>(par + n);
#pragma unroll
    for (int k = 0; k < 3; ++k) soa[uint64_t(k) * n + i] = means[3 * i + k];
#pragma unroll
    for (int k = 0; k < 3; ++k) soa[uint64_t(3 + k) * n + i] = scales[3 * i + k];
#pragma unroll
    for (int k = 0; k < 4; ++k) soa[uint64_t(6 + k) * n + i] = quats[4 * i + k];
    soa[10 * n + i] = opac[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) soa[uint64_t(11 + k) * n + i] = cols[3 * i + k];
    parent[i] = par[i];
    leaf[i] = lf[i];
}

// Last index holding a non-leaf (for DevTree::leaf_begin) and max_i |m_i|_1
// in double (for the FP32 leaf pre-test's magnitude bound); positive doubles
// order like their bit patterns, so atomicMax on the bits is exact.
__global__ void k_tree_extents(const float* __restrict__ soa, const uint8_t* __restrict__ leaf,
                               uint64_t n, unsigned long long* last_nonleaf_plus1,
                               unsigned long long* max_l1_bits) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long ln = 0, mb = 0;
    if (i < n) {
        if (!leaf[i]) ln = i + 1;
        const double l1 = fabs(double(soa[i])) + fabs(double(soa[n + i])) + fabs(double(soa[2 * n + i]));
        mb = __double_as_longlong(l1);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, ln, off);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, mb, off);
        ln = a > ln ? a : ln;
        mb = b > mb ? b : mb;
    }
    if ((threadIdx.x & 31) == 0) {
        if (ln) atomicMax(last_nonleaf_plus1, ln);
        if (mb) atomicMax(max_l1_bits, mb);
    }
}

void launch_tree_extents(const float* soa, const uint8_t* leaf, uint64_t n,
                         unsigned long long* out2, cudaStream_t s) {
    cudaMemsetAsync(out2, 0, 16, s);
    if (n) k_tree_extents<<<unsigned((n + 255) / 256), 256, 0, s>>>(soa, leaf, n, out2, out2 + 1);
}

void launch_validate_nodes(const float* soa, const uint32_t* parent, const uint8_t* leaf,
                           uint8_t* has_child, uint64_t n, const uint64_t* level_begin,
                           int n_levels, uint16_t* mask, unsigned long long* n_bad,
                           cudaStream_t s) {
    if (n == 0) return;
    const unsigned grid = unsigned((n + 255) / 256);
    cudaMemsetAsync(has_child, 0, n, s);
    k_has_child<<<grid, 256, 0, s>>>(parent, n, has_child);
    k_validate_nodes<<<grid, 256, 0, s>>>(soa, parent, leaf, has_child, n, level_begin, n_levels,
                                          mask, n_bad);
}

void launch_deinterleave(const uint8_t* payload, uint64_t n, float* soa, uint32_t* parent,
                         uint8_t* leaf, cudaStream_t s) {
    if (n) k_deinterleave<<<unsigned((n + 255) / 256), 256, 0, s>>>(payload, n, soa, parent, leaf);
}

}  // namespace fgs
