// pdl.cuh -- programmatic dependent launch for the per-frame kernel chain.
//
// A frame is a chain of stream-ordered kernels.  Launched with the
// programmatic-stream-serialization attribute, kernel N+1's CTAs may be
// scheduled while kernel N drains (every CTA of N calls pdl_trigger() on
// entry), and block in pdl_wait() -- griddepcontrol.wait: until N has
// completed and its memory is visible -- before touching N's outputs.  The
// launch latency and the tail of N overlap instead of adding up.  Kernels
// launched without the attribute return from pdl_wait() at once.
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <set>
#include <utility>

#ifndef USE_PDL
#define USE_PDL 1
#endif

namespace fgs {

__device__ __forceinline__ void pdl_wait() {
#if USE_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if USE_PDL
    asm volatile("griddepcontrol.launch_dependents;" :::);
#endif
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
#if USE_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
#else
    kernel<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
#endif
}

// Raises a kernel's dynamic shared-memory cap (default 48 KB) to `bytes`,
// once per (kernel, device).  Only the cap changes: occupancy follows the
// dynamic size of each launch.
template <typename... KArgs>
inline void opt_in_smem(void (*kernel)(KArgs...), int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (done.insert({reinterpret_cast<const void*>(kernel), dev}).second)
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace fgs
