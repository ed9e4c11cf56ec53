// The rest of a training step on the GPU (sm_100a): the loss terms of total_loss
// (proj/src/losses.cpp, ssim.cpp) with their gradient dL/dI, the opacity decay
// term (pipeline.cpp:47-52, 82-88) and the Adan / Adam update (optimizer.cpp).
//
// Precision and order: f64 throughout, like the reference.  Sums that the
// reference folds row by row (fold_partials, common.hpp:70-74) are formed the
// same way -- one thread per row summing along x, then one thread folding the
// rows in order -- so on identical inputs the loss values match the reference
// build to the last bit or two; the SSIM blurs are the reference's separable
// 11-tap correlations with zero extension (ssim.cpp:29-62).  The opacity mean is
// a fixed-shape tree reduction (deterministic, not the reference's sequential
// order).  The loss kernels are HBM-bound elementwise / stencil passes.
#include <cmath>
#include <vector>

#include "context.h"
#include "kernels.cuh"

namespace holo_cuda {

namespace {

constexpr int kWin = 11, kHalf = 5;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

__constant__ double c_win[kWin];

// ---- pointwise loss rows: (I - I_gt)^2 weighted by 1 + m^2 + b^2 (recon) or 1 (mse)
template <bool PLAIN>
__global__ void k_loss_rows(const double* __restrict__ I, const double* __restrict__ G,
                            const double* __restrict__ masks, int C, int H, int W, int L, double gscale,
                            double* __restrict__ rows, double* __restrict__ grad) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;  // row over L * C * H
    if (r >= L * C * H) return;
    const int l = r / (C * H);
    const int y = r % H;
    const size_t off = static_cast<size_t>(r) * W;
    const double* a = I + off;
    const double* b = G + off;
    const double* m = PLAIN ? nullptr : masks + (static_cast<size_t>(l) * H + y) * W;
    double* g = grad ? grad + off : nullptr;
    double acc = 0.0;
    for (int x = 0; x < W; ++x) {
        const double e = a[x] - b[x];
        const double weight = PLAIN ? 1.0 : 1.0 + m[x] * m[x] + b[x] * b[x];
        acc += weight * e * e;
        if (g) g[x] += gscale * weight * e;
    }
    rows[r] = acc;
}

// sum of n values in order (fold_partials), one thread: out = mul * sum / div
__global__ void k_fold(const double* __restrict__ v, int n, double mul, double div, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += v[i];
    *out = mul * acc / div;
}

__global__ void k_fill(double* p, int n, double v) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = v;
}

// ---- SSIM (ssim.cpp:64-147), one (plane, channel) image pair at a time
// horizontal 11-tap correlations of x, y, x^2, y^2, x y (zero extension)
__global__ void k_blur_h5(const double* __restrict__ x, const double* __restrict__ y, int W, int H,
                          double* __restrict__ out /* 5 planes */) {
    const size_t P = static_cast<size_t>(W) * H;
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= P) return;
    const int px = static_cast<int>(i % W);
    const size_t row = i - px;
    const int k0 = max(0, kHalf - px), k1 = min(kWin, W + kHalf - px);
    double s[5] = {0, 0, 0, 0, 0};
    for (int k = k0; k < k1; ++k) {
        const double w = c_win[k];
        const double xv = x[row + px + k - kHalf], yv = y[row + px + k - kHalf];
        s[0] += w * xv;
        s[1] += w * yv;
        s[2] += w * (xv * xv);
        s[3] += w * (yv * yv);
        s[4] += w * (xv * yv);
    }
    for (int q = 0; q < 5; ++q) out[q * P + i] = s[q];
}

// horizontal correlation of `n` planes
__global__ void k_blur_h(const double* __restrict__ in, int W, int H, int n, double* __restrict__ out) {
    const size_t P = static_cast<size_t>(W) * H;
    const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (t >= P * n) return;
    const size_t i = t % P, base = t - i;
    const int px = static_cast<int>(i % W);
    const size_t row = base + i - px;
    const int k0 = max(0, kHalf - px), k1 = min(kWin, W + kHalf - px);
    double acc = 0.0;
    for (int k = k0; k < k1; ++k) acc += c_win[k] * in[row + px + k - kHalf];
    out[t] = acc;
}

// vertical correlation of `n` planes
__global__ void k_blur_v(const double* __restrict__ in, int W, int H, int n, double* __restrict__ out) {
    const size_t P = static_cast<size_t>(W) * H;
    const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (t >= P * n) return;
    const size_t i = t % P, base = t - i;
    const int py = static_cast<int>(i / W), px = static_cast<int>(i % W);
    const int k0 = max(0, kHalf - py), k1 = min(kWin, H + kHalf - py);
    double acc = 0.0;
    for (int k = k0; k < k1; ++k) acc += c_win[k] * in[base + static_cast<size_t>(py + k - kHalf) * W + px];
    out[t] = acc;
}

// SSIM map over the interior window centres; gradient maps (zero outside)
__global__ void k_ssim_map(const double* __restrict__ mom /* mx my qx qy qxy */, int W, int H, int want_grad,
                           double* __restrict__ smap, double* __restrict__ gmaps /* gmu gqx gqxy */) {
    const size_t P = static_cast<size_t>(W) * H;
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= P) return;
    const int py = static_cast<int>(i / W), px = static_cast<int>(i % W);
    const bool valid = px >= kHalf && px < W - kHalf && py >= kHalf && py < H - kHalf;
    double s = 0.0, gmu = 0.0, gqx = 0.0, gqxy = 0.0;
    if (valid) {
        const double ux = mom[i], uy = mom[P + i];
        const double vxv = mom[2 * P + i] - ux * ux;
        const double vyv = mom[3 * P + i] - uy * uy;
        const double vxy = mom[4 * P + i] - ux * uy;
        const double a1 = 2.0 * ux * uy + kC1;
        const double a2 = 2.0 * vxy + kC2;
        const double b1 = ux * ux + uy * uy + kC1;
        const double b2 = vxv + vyv + kC2;
        const double d = b1 * b2;
        s = (a1 * a2) / d;
        if (want_grad) {
            gmu = (2.0 * uy * (a2 - a1) - s * 2.0 * ux * (b2 - b1)) / d;
            gqx = -s / b2;
            gqxy = 2.0 * a1 / d;
        }
    }
    smap[i] = s;
    if (want_grad) {
        gmaps[i] = gmu;
        gmaps[P + i] = gqx;
        gmaps[2 * P + i] = gqxy;
    }
}

// row sums of the SSIM map over the valid columns, one thread per valid row
__global__ void k_ssim_rows(const double* __restrict__ smap, int W, int H, double* __restrict__ rows) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int nrows = H - 2 * kHalf;
    if (r >= nrows) return;
    const double* s = smap + static_cast<size_t>(r + kHalf) * W;
    double acc = 0.0;
    for (int x = kHalf; x < W - kHalf; ++x) acc += s[x];
    rows[r] = acc;
}

// grad -= scale * (inv_n (t1 + 2 x t2 + y t3))
__global__ void k_ssim_grad(const double* __restrict__ t /* t1 t2 t3 */, const double* __restrict__ x,
                            const double* __restrict__ y, size_t P, double inv_n, double scale,
                            double* __restrict__ grad) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= P) return;
    grad[i] -= scale * (inv_n * (t[i] + 2.0 * x[i] * t[P + i] + y[i] * t[2 * P + i]));
}

__global__ void k_f32_to_f64(const float* __restrict__ in, double* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<double>(in[i]);
}

__global__ void k_f64_to_f32(const double* __restrict__ in, float* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<float>(in[i]);
}

__device__ __forceinline__ double sigmoid_ref(double x) {  // common.hpp:32-40
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    const double e = exp(x);
    return e / (1.0 + e);
}

// opacity decay: sum of sigmoids (per-block partials, fixed shape) and, with
// grads, opacity_logits += w s (1 - s)  (pipeline.cpp:82-88)
__global__ void __launch_bounds__(256) k_opacity(const double* __restrict__ logits, size_t n, double w,
                                                 double* __restrict__ partials, double* __restrict__ gopac) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (size_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * 256) {
        const double s = sigmoid_ref(logits[i]);
        acc += s;
        if (gopac) gopac[i] += w * s * (1.0 - s);
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int d = 128; d > 0; d >>= 1) {
        if (threadIdx.x < d) sh[threadIdx.x] += sh[threadIdx.x + d];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

// ---- optimizer (optimizer.cpp:70-100)
__global__ void k_nonfinite(const double* __restrict__ g, size_t n, unsigned* flag) {
    bool bad = false;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        bad = bad || !isfinite(g[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

__global__ void k_adaptive_update(double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m,
                                  double* __restrict__ v, double* __restrict__ nn, double* __restrict__ prev, size_t n,
                                  double lr, double b1, double b2, double b3, double bc1, double bc2, double bc3,
                                  double eps, int first, int adam) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double gi = g[i];
        if (adam) {
            m[i] = b1 * m[i] + (1.0 - b1) * gi;
            nn[i] = b2 * nn[i] + (1.0 - b2) * gi * gi;
            p[i] -= lr * (m[i] / bc1) / (sqrt(nn[i] / bc2) + eps);
            continue;
        }
        const double diff = first ? 0.0 : gi - prev[i];
        const double upd = gi + b2 * diff;
        m[i] = b1 * m[i] + (1.0 - b1) * gi;
        v[i] = b2 * v[i] + (1.0 - b2) * diff;
        nn[i] = b3 * nn[i] + (1.0 - b3) * upd * upd;
        prev[i] = gi;
        const double num = m[i] / bc1 + b2 * (v[i] / bc2);
        p[i] -= lr * num / (sqrt(nn[i] / bc3) + eps);
    }
}

// GaussianScene::renormalize (scene.cpp:34-47)
__global__ void k_renormalize(double* __restrict__ rot, double* __restrict__ amp, size_t n) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double* q = rot + 4 * i;
    const double norm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (norm > 1e-12) {
        for (int k = 0; k < 4; ++k) q[k] /= norm;
    } else {
        q[0] = 1.0;
        q[1] = q[2] = q[3] = 0.0;
    }
    for (int c = 0; c < 3; ++c) amp[3 * i + c] = fmax(amp[3 * i + c], 0.0);
}

unsigned blocks_for(size_t n, unsigned cap = 8192) {
    const size_t b = (n + 255) / 256;
    return static_cast<unsigned>(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace

// loss_recon / loss_mse + loss_ssim + psnr over device f64 stacks [L][C][H][W]
// (masks [L][H][W]); grad (optional, zeroed by the caller) accumulates dL/dI.
// d_out[0] = recon, d_out[1 + l] = mean SSIM of plane l, d_out[1 + L + l] =
// the mse of plane l; the host finishes the scalar algebra.
void losses_gpu(holo_ctx* ctx, const double* I, const double* G, const double* masks, int L, int C, int H, int W,
                bool plain, bool with_ssim, double lambda_ssim, double* grad, double* d_out) {
    const size_t n = static_cast<size_t>(C) * H * W, P = static_cast<size_t>(H) * W;
    if (with_ssim && (W < kWin || H < kWin))
        throw Error(HOLO_ERR_CONFIG, "ssim needs images at least 11 pixels in each dimension");
    static bool win_set = false;
    if (!win_set) {  // ssim.cpp:16-26
        double w[kWin], sum = 0.0;
        for (int i = 0; i < kWin; ++i) {
            const double d = i - kHalf;
            w[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            sum += w[i];
        }
        for (double& v : w) v /= sum;
        HC_CUDA(cudaMemcpyToSymbol(c_win, w, sizeof w));
        win_set = true;
    }
    const int rows_n = L * C * H;
    double* rows = static_cast<double*>(ctx->buffer("loss_rows", sizeof(double) * rows_n));
    double* prow = static_cast<double*>(ctx->buffer("psnr_rows", sizeof(double) * rows_n));
    double* lsum = static_cast<double*>(ctx->buffer("loss_plane", sizeof(double) * L));
    const double inv_l = 1.0 / static_cast<double>(L), inv_n = 1.0 / static_cast<double>(n);
    const unsigned rb = (rows_n + 127) / 128;
    // recon / mse (losses.cpp:28-94): every plane has the same n, so one pass
    if (plain)
        k_loss_rows<true><<<rb, 128, 0, ctx->stream>>>(I, G, masks, C, H, W, L, 2.0 * inv_l * inv_n, rows, grad);
    else
        k_loss_rows<false><<<rb, 128, 0, ctx->stream>>>(I, G, masks, C, H, W, L, 2.0 * inv_l * inv_n, rows, grad);
    HC_LAUNCHED(ctx);
    // psnr (losses.cpp:113-132): plain squared-error rows
    k_loss_rows<true><<<rb, 128, 0, ctx->stream>>>(I, G, nullptr, C, H, W, L, 0.0, prow, nullptr);
    HC_LAUNCHED(ctx);
    for (int l = 0; l < L; ++l) {
        const size_t ro = static_cast<size_t>(l) * C * H;
        k_fold<<<1, 32, 0, ctx->stream>>>(rows + ro, C * H, inv_l * inv_n, 1.0, lsum + l);
        HC_LAUNCHED(ctx);
        k_fold<<<1, 32, 0, ctx->stream>>>(prow + ro, C * H, 1.0, static_cast<double>(n), d_out + 1 + L + l);
        HC_LAUNCHED(ctx);
    }
    k_fold<<<1, 32, 0, ctx->stream>>>(lsum, L, 1.0, 1.0, d_out);
    HC_LAUNCHED(ctx);

    if (!with_ssim) {  // the SSIM term left out: mean SSIM 1 contributes 0
        k_fill<<<1, 32, 0, ctx->stream>>>(d_out + 1, L, 1.0);
        HC_LAUNCHED(ctx);
        return;
    }
    // ssim (losses.cpp:96-111, ssim.cpp:64-147): lambda / L (1 - mean SSIM) per plane
    const int vrows = H - 2 * kHalf;
    const size_t n_valid = static_cast<size_t>(W - 2 * kHalf) * vrows * C;
    const double inv_valid = 1.0 / static_cast<double>(n_valid);
    double* mom = static_cast<double*>(ctx->buffer("ssim_mom", sizeof(double) * 5 * P));
    double* scratch = static_cast<double*>(ctx->buffer("ssim_scratch", sizeof(double) * 5 * P));
    double* smap = static_cast<double*>(ctx->buffer("ssim_map", sizeof(double) * P));
    double* gmaps = grad ? static_cast<double*>(ctx->buffer("ssim_gmaps", sizeof(double) * 3 * P)) : nullptr;
    double* srows = static_cast<double*>(ctx->buffer("ssim_rows", sizeof(double) * vrows));
    double* ssum = static_cast<double*>(ctx->buffer("ssim_sum", sizeof(double) * C));
    const unsigned pb = blocks_for(P, 1u << 30);
    for (int l = 0; l < L; ++l) {
        for (int c = 0; c < C; ++c) {
            const size_t off = (static_cast<size_t>(l) * C + c) * P;
            k_blur_h5<<<pb, 256, 0, ctx->stream>>>(I + off, G + off, W, H, scratch);
            HC_LAUNCHED(ctx);
            k_blur_v<<<blocks_for(5 * P, 1u << 30), 256, 0, ctx->stream>>>(scratch, W, H, 5, mom);
            HC_LAUNCHED(ctx);
            k_ssim_map<<<pb, 256, 0, ctx->stream>>>(mom, W, H, grad != nullptr, smap, gmaps);
            HC_LAUNCHED(ctx);
            k_ssim_rows<<<(vrows + 127) / 128, 128, 0, ctx->stream>>>(smap, W, H, srows);
            HC_LAUNCHED(ctx);
            k_fold<<<1, 32, 0, ctx->stream>>>(srows, vrows, 1.0, 1.0, ssum + c);
            HC_LAUNCHED(ctx);
            if (grad) {
                k_blur_h<<<blocks_for(3 * P, 1u << 30), 256, 0, ctx->stream>>>(gmaps, W, H, 3, scratch);
                HC_LAUNCHED(ctx);
                k_blur_v<<<blocks_for(3 * P, 1u << 30), 256, 0, ctx->stream>>>(scratch, W, H, 3, mom);
                HC_LAUNCHED(ctx);
                k_ssim_grad<<<pb, 256, 0, ctx->stream>>>(mom, I + off, G + off, P, inv_valid,
                                                         lambda_ssim / static_cast<double>(L), grad + off);
                HC_LAUNCHED(ctx);
            }
        }
        // channels folded in order, / n_valid (ssim.cpp:123, 146)
        k_fold<<<1, 32, 0, ctx->stream>>>(ssum, C, 1.0, static_cast<double>(n_valid), d_out + 1 + l);
        HC_LAUNCHED(ctx);
    }
}

double opacity_term(holo_ctx* ctx, const double* logits, size_t n, double lambda, double* gopac) {
    if (n == 0 || lambda == 0.0) return 0.0;
    const unsigned nb = blocks_for(n, 4096);
    double* part = static_cast<double*>(ctx->buffer("opac_part", sizeof(double) * nb));
    k_opacity<<<nb, 256, 0, ctx->stream>>>(logits, n, lambda / static_cast<double>(n), part, gopac);
    HC_LAUNCHED(ctx);
    std::vector<double> h(nb);
    HC_CUDA(cudaMemcpyAsync(h.data(), part, sizeof(double) * nb, cudaMemcpyDeviceToHost, ctx->stream));
    HC_CUDA(cudaStreamSynchronize(ctx->stream));
    double s = 0.0;
    for (double v : h) s += v;
    return lambda * s / static_cast<double>(n);
}

void f32_to_f64(holo_ctx* ctx, const float* in, double* out, size_t n) {
    k_f32_to_f64<<<blocks_for(n), 256, 0, ctx->stream>>>(in, out, n);
    HC_LAUNCHED(ctx);
}

void f64_to_f32(holo_ctx* ctx, const double* in, float* out, size_t n) {
    k_f64_to_f32<<<blocks_for(n), 256, 0, ctx->stream>>>(in, out, n);
    HC_LAUNCHED(ctx);
}

bool grads_finite(holo_ctx* ctx, const double* const* g, const size_t* n, int groups) {
    unsigned* flag = static_cast<unsigned*>(ctx->buffer("nonfinite", sizeof(unsigned)));
    HC_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned), ctx->stream));
    for (int k = 0; k < groups; ++k)
        if (g[k] && n[k]) {
            k_nonfinite<<<blocks_for(n[k], 2048), 256, 0, ctx->stream>>>(g[k], n[k], flag);
            HC_LAUNCHED(ctx);
        }
    unsigned h = 0;
    HC_CUDA(cudaMemcpyAsync(&h, flag, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    HC_CUDA(cudaStreamSynchronize(ctx->stream));
    return h == 0;
}

void adaptive_update(holo_ctx* ctx, double* p, const double* g, double* m, double* v, double* nn, double* prev,
                     size_t n, double lr, long long step, double b1, double b2, double b3, double eps, bool adam) {
    if (n == 0) return;
    const double bc1 = 1.0 - std::pow(b1, static_cast<double>(step));
    const double bc2 = 1.0 - std::pow(b2, static_cast<double>(step));
    const double bc3 = 1.0 - std::pow(b3, static_cast<double>(step));
    k_adaptive_update<<<blocks_for(n), 256, 0, ctx->stream>>>(p, g, m, v, nn, prev, n, lr, b1, b2, b3, bc1, bc2, bc3,
                                                              eps, step == 1 ? 1 : 0, adam ? 1 : 0);
    HC_LAUNCHED(ctx);
}

void renormalize_scene(holo_ctx* ctx, double* rot, double* amp, size_t n) {
    if (n == 0) return;
    k_renormalize<<<blocks_for(n, 1u << 30), 256, 0, ctx->stream>>>(rot, amp, n);
    HC_LAUNCHED(ctx);
}

}  // namespace holo_cuda
