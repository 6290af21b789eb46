// Issue rate of packed FP32x2 FMA (FFMA2) vs scalar FFMA on sm_100a: 8
// independent chains per thread, 148 x 8 CTAs of 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__global__ void k1(float* out, int iters, float s) {
    float v[8];
    for (int j = 0; j < 8; ++j) v[j] = threadIdx.x * 1e-3f + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __fmaf_rn(v[j], s, 0.5f);
    float t = 0;
    for (int j = 0; j < 8; ++j) t += v[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k2(float* out, int iters, float s) {
    unsigned long long v[8], ss, h;
    asm("mov.b64 %0, {%1,%1};" : "=l"(ss) : "f"(s));
    asm("mov.b64 %0, {%1,%1};" : "=l"(h) : "f"(0.5f));
    for (int j = 0; j < 8; ++j) {
        float a = threadIdx.x * 1e-3f + j;
        asm("mov.b64 %0, {%1,%1};" : "=l"(v[j]) : "f"(a));
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = fma2(v[j], ss, h);
    float t = 0;
    for (int j = 0; j < 8; ++j) {
        float a, b;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v[j]));
        t += a + b;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
    float* o;
    cudaMalloc(&o, 148 * 8 * 256 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        float ms1, ms2;
        cudaEventRecord(a);
        k1<<<148 * 8, 256>>>(o, iters, 0.999f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms1, a, b);
        cudaEventRecord(a);
        k2<<<148 * 8, 256>>>(o, iters, 0.999f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms2, a, b);
        const double n = 148.0 * 8 * 256 * iters * 8;
        printf("FFMA  %.1f Ginstr/s (%.2f TFLOP/s)\nFFMA2 %.1f Ginstr/s (%.2f TFLOP/s)\n",
               n / ms1 / 1e6, 2 * n / ms1 / 1e9, n / ms2 / 1e6, 4 * n / ms2 / 1e9);
    }
}
