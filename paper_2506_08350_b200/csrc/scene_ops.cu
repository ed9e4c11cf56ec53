// Device-side scene partitioning for plane-sharded groups (group.cu).
//
// Under hard assignment a Gaussian contributes to one plane only: the argmax of its
// plane logits, ties and NaN to the lower index (ste_assign, scene.cpp:132-152;
// the same strict '>' scan as k_preprocess).  A rank that owns planes [pb, pe)
// keeps exactly the Gaussians whose plane falls there, in their original order, so
// every bucket's (depth, index) order -- and hence its layers and partial spectrum
// -- is that of the full scene (rasterizer.cpp:221-224).  The subset is formed on
// the device from the uploaded scene: a flag per Gaussian, an exclusive scan, and a
// stable scatter of the seven f64 arrays.
#include <algorithm>
#include "kernels.cuh"

namespace holo_cuda {

namespace {

__global__ void k_plane_keep(const double* __restrict__ logits, size_t n, int L, int pb, int pe,
                             unsigned* __restrict__ keep) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double* lg = logits + i * L;
        int best = 0;
        double top = lg[0];
        for (int l = 1; l < L; ++l) {
            const double v = lg[l];
            if (v > top) {
                top = v;
                best = l;
            }
        }
        keep[i] = (best >= pb && best < pe) ? 1u : 0u;
    }
}

struct SceneCols {
    const double* src[7];
    double* dst[7];
    int width[7];
};

// one thread per (Gaussian, array) row; rows are 1..L doubles wide
__global__ void k_scene_scatter(SceneCols cols, size_t n, const unsigned* __restrict__ keep,
                                const unsigned* __restrict__ offs) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        if (!keep[i]) continue;
        const size_t j = offs[i];
#pragma unroll
        for (int a = 0; a < 7; ++a) {
            const int w = cols.width[a];
            const double* s = cols.src[a] + i * w;
            double* d = cols.dst[a] + j * w;
            for (int k = 0; k < w; ++k) d[k] = s[k];
        }
    }
}

}  // namespace

size_t scene_keep_planes(holo_ctx* ctx, const double* const src[7], double* const dst[7], size_t n, int L, int pb,
                         int pe) {
    if (n == 0) return 0;
    unsigned* keep = static_cast<unsigned*>(ctx->buffer("subset_keep", sizeof(unsigned) * (n + 1)));
    unsigned* offs = static_cast<unsigned*>(ctx->buffer("subset_offs", sizeof(unsigned) * (n + 1)));
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 8 * 148));
    k_plane_keep<<<blocks, 256, 0, ctx->stream>>>(src[6], n, L, pb, pe, keep);
    HC_LAUNCHED(ctx);
    exclusive_scan_u32(ctx, keep, offs, static_cast<long long>(n), nullptr);
    SceneCols cols{};
    const int width[7] = {3, 4, 3, 3, 1, 3, L};
    for (int a = 0; a < 7; ++a) {
        cols.src[a] = src[a];
        cols.dst[a] = dst[a];
        cols.width[a] = width[a];
    }
    k_scene_scatter<<<blocks, 256, 0, ctx->stream>>>(cols, n, keep, offs);
    HC_LAUNCHED(ctx);
    unsigned count = 0;
    HC_CUDA(cudaMemcpyAsync(&count, offs + n, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
    HC_CUDA(cudaStreamSynchronize(ctx->stream));
    return count;
}

namespace {
// make_target_from_scene's masks (pipeline.cpp:106-124): pixel p belongs to the
// plane whose rasterised amplitude sum_c |layer_c(p)| (f64, of the fp32 layer
// widened exactly as the drop-in returns it) is the strict maximum, the first
// such plane on ties; untouched pixels (all sums 0) stay unmasked.
__global__ void k_plane_masks(const cx<float>* __restrict__ layers, int L, int C, size_t P,
                              double* __restrict__ masks) {
    for (size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; p < P;
         p += static_cast<size_t>(gridDim.x) * blockDim.x) {
        int best = -1;
        double best_amp = 0.0;
        for (int l = 0; l < L; ++l) {
            double amp = 0.0;
            for (int c = 0; c < C; ++c) {
                const cx<float> v = layers[(static_cast<size_t>(l) * C + c) * P + p];
                amp += hypot(static_cast<double>(v.x), static_cast<double>(v.y));
            }
            if (amp > best_amp) {
                best_amp = amp;
                best = l;
            }
        }
        for (int l = 0; l < L; ++l) masks[static_cast<size_t>(l) * P + p] = l == best ? 1.0 : 0.0;
    }
}
}  // namespace

void plane_masks(holo_ctx* ctx, const cx<float>* layers, int L, int C, size_t P, double* masks) {
    if (P == 0 || L == 0) return;
    const unsigned grid = static_cast<unsigned>(std::min<size_t>((P + 255) / 256, 8 * 148));
    k_plane_masks<<<grid, 256, 0, ctx->stream>>>(layers, L, C, P, masks);
    HC_LAUNCHED(ctx);
}

}  // namespace holo_cuda
