// HBM bandwidth of column-strip access: [F][H][W] float2, each CTA copies an
// NB-column strip of H rows (NB*8-byte segments at a W*8-byte stride), versus a
// contiguous copy of the same bytes.
#include <cstdio>
#include <cuda_runtime.h>
template <int NB>
__global__ void strip(const float2* __restrict__ in, float2* __restrict__ out, int W, int H) {
    const int x0 = blockIdx.x * NB;
    const size_t base = (size_t)blockIdx.y * H * W;
    for (int t = threadIdx.x; t < H * NB; t += blockDim.x) {
        const int i = t / NB, b = t % NB;
        const size_t at = base + (size_t)i * W + x0 + b;
        out[at] = in[at];
    }
}
__global__ void contig(const float4* __restrict__ in, float4* __restrict__ out, size_t n) {
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) out[t] = in[t];
}
int main() {
    const int W = 1920, H = 1080, F = 24;
    const size_t n = (size_t)F * H * W;
    float2 *a, *b;
    cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8);
    cudaMemset(a, 0, n * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(e0); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
        printf("%-28s %.3f ms  %.0f GB/s\n", name, ms, 2.0 * n * 8 / ms / 1e6);
    };
    run("contiguous", [&] { contig<<<148 * 8, 512>>>((const float4*)a, (float4*)b, n / 2); });
    run("strip NB=4", [&] { strip<4><<<dim3(W / 4, F), 512>>>(a, b, W, H); });
    run("strip NB=8", [&] { strip<8><<<dim3(W / 8, F), 512>>>(a, b, W, H); });
    run("strip NB=16", [&] { strip<16><<<dim3(W / 16, F), 512>>>(a, b, W, H); });
    run("strip NB=32", [&] { strip<32><<<dim3(W / 32, F), 512>>>(a, b, W, H); });
    return 0;
}
