// brute_force_forward (rasterizer.cpp:265-315) on the GPU: the same per-pixel
// math as the tiled compositing, with no tiles, no support-radius culling and no
// early termination -- every valid Gaussian of the plane, in the global (zc, index)
// order, at every pixel.  The reference keeps it as the equivalence oracle of its
// tiled pass ("tiled pass equals brute force bitwise when termination is off",
// test_rasterizer.cpp:244-255); here it evaluates each entry with the staged record
// and the instruction sequence of k_composite (raster_eval.cuh), relative to the
// pixel's tile origin as k_composite does, so the two agree bit for bit whenever
// the reference's do.  Test-oracle throughput: one thread per pixel walks all N.
#include "raster_eval.cuh"

namespace holo_cuda {

namespace {

template <int C>
__global__ void k_brute(const GRec* __restrict__ rec, const int* __restrict__ order, int n_order,
                        const int* __restrict__ plane_of, const double* __restrict__ rho, int L, int W, int H,
                        int tile, int soft, int gate_open, float alpha_floor, int floor_positive, float clamp,
                        cx<float>* __restrict__ layers) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x;
    const int py = blockIdx.y * blockDim.y + threadIdx.y;
    const int l = blockIdx.z;
    if (px >= W || py >= H) return;
    const int px0 = (px / tile) * tile, py0 = (py / tile) * tile;
    const float fx = static_cast<float>(px - px0) + 0.5f, fy = static_cast<float>(py - py0) + 0.5f;
    const float thr = floor_positive ? alpha_floor : 0.0f;
    const float eps = 0.0f;  // no early termination
    float T = 1.0f;
    cx<float> acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = mk(0.0f, 0.0f);
    for (int k = 0; k < n_order; ++k) {
        const int g = order[k];
        float alpha;
        if (soft) {
            const double rv = rho[static_cast<size_t>(g) * L + l];
            if (!(rv > 0.0)) continue;  // soft gate 0 (rasterizer.cpp:290)
            alpha = static_cast<float>(static_cast<double>(rec[g].alpha) * rv);
        } else {
            if (!gate_open || plane_of[g] != l) continue;  // one-hot rho vs plane_eps
            alpha = rec[g].alpha;
        }
        Staged st;
        float4 box;
        stage_entry(rec[g], px0, py0, alpha, st, box);
        float4 B0;
        const float al0 = eval_alpha(&st, fx, fy, clamp, B0);
        const bool acc0 = (al0 > thr) && (T >= eps);
        const float w0 = acc0 ? al0 * T : 0.0f;
        blend<C>(&st, B0, w0, acc);
        T -= w0;
    }
    const size_t P = static_cast<size_t>(W) * H;
    const size_t pix = static_cast<size_t>(py) * W + px;
#pragma unroll
    for (int c = 0; c < C; ++c) layers[(static_cast<size_t>(l) * C + c) * P + pix] = acc[c];
}

}  // namespace

void brute_force(holo_ctx* ctx, const GRec* rec, const int* order, int n_order, const int* plane_of,
                 const double* rho, int L, int C, int W, int H, int tile, bool soft, bool gate_open,
                 float alpha_floor, bool floor_positive, float clamp, cx<float>* layers) {
    const dim3 block(16, 16);
    const dim3 grid((W + 15) / 16, (H + 15) / 16, L);
    switch (C) {
#define HB_C(CC)                                                                                                  \
    case CC:                                                                                                      \
        k_brute<CC><<<grid, block, 0, ctx->stream>>>(rec, order, n_order, plane_of, rho, L, W, H, tile, soft,    \
                                                     gate_open, alpha_floor, floor_positive, clamp, layers);      \
        break;
        HB_C(1)
        HB_C(2)
        HB_C(3)
#undef HB_C
        default:
            throw Error(HOLO_ERR_CONFIG, "render supports 1 to 3 wavelength channels");
    }
    HC_LAUNCHED(ctx);
}

}  // namespace holo_cuda
