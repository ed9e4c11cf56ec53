// Throughput of packed fp32x2 (FFMA2 / FADD2) versus scalar FFMA on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__global__ void k_scalar(float* out, int iters, float s) {
    float a[8];
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 0.001f + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], s, 0.5f);
    float t = 0; for (int j = 0; j < 8; ++j) t += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_packed(float* out, int iters, float s) {
    unsigned long long a[4];
    for (int j = 0; j < 4; ++j) a[j] = pk(threadIdx.x * 0.001f + j, j + 0.5f);
    const unsigned long long ss = pk(s, s), hh = pk(0.5f, 0.5f);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(ss), "l"(hh));
    float t = 0;
    for (int j = 0; j < 4; ++j) { float u, v; asm("mov.b64 {%0, %1}, %2;" : "=f"(u), "=f"(v) : "l"(a[j])); t += u + v; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
    float* d; cudaMalloc(&d, 148 * 8 * 1024 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); k_scalar<<<blocks, threads>>>(d, iters, 0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * iters * (double)blocks * threads;
        printf("scalar FFMA : %.2f ms  %.1f TFLOP/s  %.2f Tinst/s(warp)\n", ms, fl / ms / 1e9, fl / 2 / 32 / ms / 1e9);
        cudaEventRecord(e0); k_packed<<<blocks, threads>>>(d, iters, 0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("packed FFMA2: %.2f ms  %.1f TFLOP/s  %.2f Tinst/s(warp)\n", ms, fl / ms / 1e9, fl / 4 / 32 / ms / 1e9);
    }
    return 0;
}
