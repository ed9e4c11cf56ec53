// Phase-only conversion on the GPU (sm_100a): the elementwise pieces of
// phase_only_loss / convert_phase_only (proj/src/phase_only.cpp:22-118).  The
// propagation around them is the f64 operator set (FFT sweeps with the transfer
// function fused into the column pass), orchestrated in capi.cu.  Fields are f64
// like the reference; the matching sums are fixed-shape tree reductions
// (deterministic run to run, not the reference's sequential fold).
#include "context.h"
#include "kernels.cuh"

namespace holo_cuda {

namespace {

constexpr int kThreads = 256;

unsigned grid_for(size_t n, unsigned cap = 1u << 20) {
    const size_t b = (n + kThreads - 1) / kThreads;
    return static_cast<unsigned>(b < cap ? (b ? b : 1) : cap);
}

// index of crop sample (c, y, x) in the (padded) grid
__device__ __forceinline__ size_t grid_index(int c, int y, int x, int w, int h, bool pad) {
    if (!pad) return (static_cast<size_t>(c) * h + y) * w + x;
    const int pw = 2 * w, ph = 2 * h;
    const int oy = (ph - h) / 2, ox = (pw - w) / 2;  // pad_center (propagation.cpp:64-72)
    return (static_cast<size_t>(c) * ph + (y + oy)) * pw + (x + ox);
}

__global__ void k_phase_field(const double* __restrict__ theta, cx<double>* __restrict__ out, int w, int h, int C,
                              bool pad) {
    const int gw = pad ? 2 * w : w, gh = pad ? 2 * h : h;
    const size_t total = static_cast<size_t>(C) * gw * gh;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int gx = static_cast<int>(i % gw);
        const int gy = static_cast<int>((i / gw) % gh);
        const int c = static_cast<int>(i / (static_cast<size_t>(gw) * gh));
        const int x = pad ? gx - (gw - w) / 2 : gx, y = pad ? gy - (gh - h) / 2 : gy;
        cx<double> v = mk(0.0, 0.0);
        if (x >= 0 && x < w && y >= 0 && y < h) {
            double s, co;
            sincos(theta[(static_cast<size_t>(c) * h + y) * w + x], &s, &co);  // std::polar(1, theta)
            v = mk(co, s);
        }
        out[i] = v;
    }
}

// one block per (plane, block-slice): partial sums of |rep - tf|^2 in a fixed tree
__global__ void __launch_bounds__(kThreads) k_phase_match(const cx<double>* __restrict__ rep,
                                                          const cx<double>* __restrict__ tf, int w, int h, int C,
                                                          bool pad, double* __restrict__ images,
                                                          double* __restrict__ partials) {
    __shared__ double sh[kThreads];
    const int l = blockIdx.y;
    const size_t n = static_cast<size_t>(C) * h * w;
    const size_t gn = pad ? 4 * n : n;
    double acc = 0.0;
    for (size_t i = blockIdx.x * static_cast<size_t>(kThreads) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * kThreads) {
        const int x = static_cast<int>(i % w), y = static_cast<int>((i / w) % h);
        const int c = static_cast<int>(i / (static_cast<size_t>(w) * h));
        const cx<double> r = rep[l * gn + grid_index(c, y, x, w, h, pad)];
        const cx<double> t = tf[l * n + i];
        const double dr = r.x - t.x, di = r.y - t.y;
        acc += dr * dr + di * di;  // std::norm
        images[l * n + i] = r.x * r.x + r.y * r.y;
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int d = kThreads / 2; d > 0; d >>= 1) {
        if (threadIdx.x < d) sh[threadIdx.x] += sh[threadIdx.x + d];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[static_cast<size_t>(l) * gridDim.x + blockIdx.x] = sh[0];
}

__global__ void k_sum_rows(const double* __restrict__ partials, int nb, int L, double* __restrict__ out) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= L) return;
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) acc += partials[static_cast<size_t>(l) * nb + b];
    out[l] = acc;
}

__global__ void k_phase_seed(cx<double>* __restrict__ rep, const cx<double>* __restrict__ tf,
                             const double* __restrict__ gi, int w, int h, int C, int L, bool pad, double inv_lm) {
    const int gw = pad ? 2 * w : w, gh = pad ? 2 * h : h;
    const size_t gn = static_cast<size_t>(C) * gw * gh, n = static_cast<size_t>(C) * w * h;
    const size_t total = gn * L;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t l = i / gn, j = i % gn;
        const int gx = static_cast<int>(j % gw);
        const int gy = static_cast<int>((j / gw) % gh);
        const int c = static_cast<int>(j / (static_cast<size_t>(gw) * gh));
        const int x = pad ? gx - (gw - w) / 2 : gx, y = pad ? gy - (gh - h) / 2 : gy;
        if (y < 0 || y >= h) continue;  // rows outside the crop are never read (pruned transforms)
        cx<double> v = mk(0.0, 0.0);
        if (x >= 0 && x < w) {
            const size_t k = l * n + (static_cast<size_t>(c) * h + y) * w + x;
            const cx<double> r = rep[i], t = tf[k];
            const double g = gi[k];
            // 2 inv_lm (rep - tf) + 2 rep gi (phase_only.cpp:87-89)
            v = mk(2.0 * inv_lm * (r.x - t.x) + 2.0 * r.x * g, 2.0 * inv_lm * (r.y - t.y) + 2.0 * r.y * g);
        }
        rep[i] = v;
    }
}

__global__ void k_phase_grad(const cx<double>* __restrict__ acc, const double* __restrict__ theta,
                             double* __restrict__ grad, int w, int h, int C, bool pad) {
    const size_t n = static_cast<size_t>(C) * h * w;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % w), y = static_cast<int>((i / w) % h);
        const int c = static_cast<int>(i / (static_cast<size_t>(w) * h));
        const cx<double> a = acc[grid_index(c, y, x, w, h, pad)];
        double s, co;
        sincos(theta[i], &s, &co);
        grad[i] = a.y * co - a.x * s;  // Im(a conj(e^{j theta})) (phase_only.cpp:97-99)
    }
}

__global__ void k_phase_arg(const cx<double>* __restrict__ P, double* __restrict__ theta, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        theta[i] = atan2(P[i].y, P[i].x);
}

__global__ void k_nonfinite_c128(const cx<double>* __restrict__ P, size_t n, unsigned* flag) {
    bool bad = false;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        bad = bad || !isfinite(P[i].x) || !isfinite(P[i].y);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

}  // namespace

void phase_field(holo_ctx* ctx, const double* theta, cx<double>* out, int w, int h, int C, bool pad) {
    const size_t total = static_cast<size_t>(C) * w * h * (pad ? 4 : 1);
    k_phase_field<<<grid_for(total), kThreads, 0, ctx->stream>>>(theta, out, w, h, C, pad);
    HC_LAUNCHED(ctx);
}

void phase_match(holo_ctx* ctx, const cx<double>* rep, const cx<double>* tf, int w, int h, int C, int L, bool pad,
                 double* images, double* plane_sums) {
    const size_t n = static_cast<size_t>(C) * w * h;
    const unsigned nb = grid_for(n, 2 * static_cast<unsigned>(ctx->sm_count));
    double* part = static_cast<double*>(ctx->buffer("po_part", sizeof(double) * nb * L));
    k_phase_match<<<dim3(nb, L), kThreads, 0, ctx->stream>>>(rep, tf, w, h, C, pad, images, part);
    HC_LAUNCHED(ctx);
    k_sum_rows<<<(L + 31) / 32, 32, 0, ctx->stream>>>(part, static_cast<int>(nb), L, plane_sums);
    HC_LAUNCHED(ctx);
}

void phase_seed(holo_ctx* ctx, cx<double>* rep, const cx<double>* tf, const double* gi, int w, int h, int C, int L,
                bool pad, double inv_lm) {
    const size_t total = static_cast<size_t>(C) * w * h * (pad ? 4 : 1) * L;
    k_phase_seed<<<grid_for(total), kThreads, 0, ctx->stream>>>(rep, tf, gi, w, h, C, L, pad, inv_lm);
    HC_LAUNCHED(ctx);
}

void phase_grad(holo_ctx* ctx, const cx<double>* acc, const double* theta, double* grad, int w, int h, int C,
                bool pad) {
    const size_t n = static_cast<size_t>(C) * w * h;
    k_phase_grad<<<grid_for(n), kThreads, 0, ctx->stream>>>(acc, theta, grad, w, h, C, pad);
    HC_LAUNCHED(ctx);
}

void phase_arg(holo_ctx* ctx, const cx<double>* P, double* theta, size_t n) {
    k_phase_arg<<<grid_for(n), kThreads, 0, ctx->stream>>>(P, theta, n);
    HC_LAUNCHED(ctx);
}

bool all_finite_c128(holo_ctx* ctx, const cx<double>* P, size_t n) {
    unsigned* flag = static_cast<unsigned*>(ctx->buffer("po_flag", sizeof(unsigned)));
    HC_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned), ctx->stream));
    k_nonfinite_c128<<<grid_for(n, 2048), kThreads, 0, ctx->stream>>>(P, n, flag);
    HC_LAUNCHED(ctx);
    unsigned hflag = 0;
    HC_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof hflag, cudaMemcpyDeviceToHost, ctx->stream));
    HC_CUDA(cudaStreamSynchronize(ctx->stream));
    return hflag == 0;
}

}  // namespace holo_cuda
