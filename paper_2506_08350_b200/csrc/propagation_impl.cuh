#pragma once
// Angular-spectrum propagation on sm_100a (templates; instantiated by propagation_f32.cu / propagation_f64.cu): batched Stockham row/column FFT
// kernels and the fused spectrum / replay column passes.
//
// Replaces proj/src/fft.cpp:33-44 (fft2/ifft2), propagation.cpp:18-123
// (build_tf, apply_tf_channel, propagate, forward_record, inverse_propagate) and
// field.cpp:5-14 (intensity).  The transfer function is never materialised on
// the render path: tf_value() evaluates it per element inside the column pass.
#include <cmath>
#include <cstring>
#include <type_traits>

#include "context.h"
#include "kernels.cuh"

namespace holo_cuda {

// ------------------------------------------------------------------ planning

#ifdef HOLO_PROPAGATION_COMMON
FftPlan plan_or_throw(int n) {
    FftPlan p;
    if (!make_plan(n, &p))
        throw Error(HOLO_ERR_CONFIG, "FFT length " + std::to_string(n) + " has a prime factor above 31");
    return p;
}
#endif

// ------------------------------------------------------------------ kernels

template <class T>
__device__ __forceinline__ cx<T> czero() {
    return mk<T>(T(0), T(0));
}

// Row FFT of nrows contiguous rows of length n; nb rows per CTA.
template <class T, int DIR>
__global__ void __launch_bounds__(256) k_rows(const cx<T>* __restrict__ in, cx<T>* __restrict__ out, int n,
                                              long long nrows, int nb, FftPlan plan, const cx<T>* __restrict__ tw,
                                              T s) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<T>* b0 = reinterpret_cast<cx<T>*>(smem_raw);
    cx<T>* b1 = b0 + static_cast<size_t>(n) * nb;
    const long long row0 = static_cast<long long>(blockIdx.x) * nb;
    const int rows = static_cast<int>(nrows - row0 < nb ? nrows - row0 : nb);
    const int tot = n * nb;
    const cx<T>* src = in + row0 * n;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) b0[t] = (t < rows * n) ? src[t] : czero<T>();
    __syncthreads();
    const cx<T>* r = fft_batch<DIR, T>(b0, b1, RowLayout{n, nb}, plan, tw);
    cx<T>* dst = out + row0 * n;
    for (int t = threadIdx.x; t < rows * n; t += blockDim.x) dst[t] = scale(r[t], s);
}

// Column FFT of batch fields [batch][h][w]; one CTA per (strip of nb columns, field).
template <class T, int DIR>
__global__ void __launch_bounds__(256) k_cols(const cx<T>* __restrict__ in, cx<T>* __restrict__ out, int w, int h,
                                              int nb, FftPlan plan, const cx<T>* __restrict__ tw, T s) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<T>* b0 = reinterpret_cast<cx<T>*>(smem_raw);
    cx<T>* b1 = b0 + static_cast<size_t>(h) * nb;
    const int x0 = blockIdx.x * nb;
    const size_t base = static_cast<size_t>(blockIdx.y) * h * w;
    const int tot = h * nb;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) {
        const int b = t % nb, i = t / nb, x = x0 + b;
        b0[t] = x < w ? in[base + static_cast<size_t>(i) * w + x] : czero<T>();
    }
    __syncthreads();
    const cx<T>* r = fft_batch<DIR, T>(b0, b1, ColLayout{h, nb}, plan, tw);
    for (int t = threadIdx.x; t < tot; t += blockDim.x) {
        const int b = t % nb, i = t / nb, x = x0 + b;
        if (x < w) out[base + static_cast<size_t>(i) * w + x] = scale(r[t], s);
    }
}

// S[c] = sum_l H_{z_l, c} . colFFT(layers[l][c]) for row-transformed layers
// [L][C][h][w].  One CTA per (strip, channel); the spectrum strip accumulates in
// shared memory in plane order, so the sum is deterministic.
// Optional (ColOpts): tftab = the transfer functions precomputed [L][C][h][w] (a
// loop that applies the same planes many times: phase-only conversion), and
// [row_lo, row_hi) = the only input rows that can be nonzero (padded fields).
template <class T>
__global__ void __launch_bounds__(256) k_col_spectrum(const cx<T>* __restrict__ layers, cx<T>* __restrict__ spec,
                                                      int w, int h, int C, int L, int nb, FftPlan plan,
                                                      const cx<T>* __restrict__ tw, const TfChan* __restrict__ tfc,
                                                      const double* __restrict__ fx, const double* __restrict__ fy,
                                                      const cx<T>* __restrict__ tftab, int row_lo, int row_hi) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<T>* b0 = reinterpret_cast<cx<T>*>(smem_raw);
    cx<T>* b1 = b0 + static_cast<size_t>(h) * nb;
    cx<T>* sacc = b1 + static_cast<size_t>(h) * nb;
    const int x0 = blockIdx.x * nb;
    const int c = blockIdx.y;
    const int tot = h * nb;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) sacc[t] = czero<T>();
    for (int l = 0; l < L; ++l) {
        const cx<T>* src = layers + (static_cast<size_t>(l) * C + c) * h * w;
        for (int t = threadIdx.x; t < tot; t += blockDim.x) {
            const int b = t % nb, i = t / nb, x = x0 + b;
            b0[t] = (x < w && i >= row_lo && i < row_hi) ? src[static_cast<size_t>(i) * w + x] : czero<T>();
        }
        __syncthreads();
        const cx<T>* r = fft_batch<-1, T>(b0, b1, ColLayout{h, nb}, plan, tw);
        const TfChan p = tfc[l * C + c];
        const cx<T>* tab = tftab ? tftab + (static_cast<size_t>(l) * C + c) * h * w : nullptr;
        for (int t = threadIdx.x; t < tot; t += blockDim.x) {
            const int b = t % nb, i = t / nb, x = x0 + b;
            if (x < w)
                sacc[t] = sacc[t] + r[t] * (tab ? tab[static_cast<size_t>(i) * w + x] : tf_value<T>(p, fx[x], fy[i]));
        }
        __syncthreads();
    }
    cx<T>* dst = spec + static_cast<size_t>(c) * h * w;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) {
        const int b = t % nb, i = t / nb, x = x0 + b;
        if (x < w) dst[static_cast<size_t>(i) * w + x] = sacc[t];
    }
}

// out[o][c] = colIFFT(M_o . S[c]) with M_o = conj(H_{z_{plane[o]}}) = H_{-z}, or 1
// when plane[o] < 0 (the hologram itself).  One CTA per (strip, channel, output).
template <class T>
__global__ void __launch_bounds__(256) k_col_replay(const cx<T>* __restrict__ spec, cx<T>* __restrict__ out,
                                                    int w, int h, int C, int nb, FftPlan plan,
                                                    const cx<T>* __restrict__ tw, const TfChan* __restrict__ tfc,
                                                    const int* __restrict__ plane_of,
                                                    const double* __restrict__ fx, const double* __restrict__ fy,
                                                    const cx<T>* __restrict__ tftab, int row_lo, int row_hi) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<T>* b0 = reinterpret_cast<cx<T>*>(smem_raw);
    cx<T>* b1 = b0 + static_cast<size_t>(h) * nb;
    const int x0 = blockIdx.x * nb;
    const int c = blockIdx.y;
    const int o = blockIdx.z;
    const int l = plane_of[o];
    const int tot = h * nb;
    const cx<T>* src = spec + static_cast<size_t>(c) * h * w;
    TfChan p;
    if (l >= 0) p = tfc[l * C + c];
    const cx<T>* tab = (tftab && l >= 0) ? tftab + (static_cast<size_t>(l) * C + c) * h * w : nullptr;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) {
        const int b = t % nb, i = t / nb, x = x0 + b;
        cx<T> v = czero<T>();
        if (x < w) {
            v = src[static_cast<size_t>(i) * w + x];
            if (l >= 0) v = v * conj(tab ? tab[static_cast<size_t>(i) * w + x] : tf_value<T>(p, fx[x], fy[i]));
        }
        b0[t] = v;
    }
    __syncthreads();
    const cx<T>* r = fft_batch<+1, T>(b0, b1, ColLayout{h, nb}, plan, tw);
    cx<T>* dst = out + (static_cast<size_t>(o) * C + c) * h * w;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) {
        const int b = t % nb, i = t / nb, x = x0 + b;
        if (x < w && i >= row_lo && i < row_hi) dst[static_cast<size_t>(i) * w + x] = r[t];
    }
}

#ifdef HOLO_PROPAGATION_COMMON
// Row IFFT of the replay staging buffer [O][C][h][w] with the render epilogues:
// output 0 (when has_holo) -> hologram * 1/(w h); the others -> intensity
// |v / (w h)|^2 (float) and optionally the replayed field v / (w h).
__global__ void __launch_bounds__(256) k_rows_epilogue(const cx<float>* __restrict__ in, int n, long long nrows,
                                                       int nb, int C, int h, int has_holo, FftPlan plan,
                                                       const cx<float>* __restrict__ tw, float s,
                                                       cx<float>* __restrict__ holo, cx<float>* __restrict__ replayed,
                                                       float* __restrict__ intens) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<float>* b0 = reinterpret_cast<cx<float>*>(smem_raw);
    cx<float>* b1 = b0 + static_cast<size_t>(n) * nb;
    const long long row0 = static_cast<long long>(blockIdx.x) * nb;
    const int rows = static_cast<int>(nrows - row0 < nb ? nrows - row0 : nb);
    const int tot = n * nb;
    const cx<float>* src = in + row0 * n;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) b0[t] = (t < rows * n) ? src[t] : czero<float>();
    __syncthreads();
    const cx<float>* r = fft_batch<+1, float>(b0, b1, RowLayout{n, nb}, plan, tw);
    const long long field_rows = static_cast<long long>(C) * h;
    for (int t = threadIdx.x; t < rows * n; t += blockDim.x) {
        const long long row = row0 + t / n;
        const int x = t % n;
        const int o = static_cast<int>(row / field_rows);
        const long long rin = row - static_cast<long long>(o) * field_rows;  // c * h + y
        const cx<float> v = scale(r[t], s);
        if (has_holo && o == 0) {
            holo[rin * n + x] = v;
        } else {
            const long long l = o - has_holo;
            const size_t at = static_cast<size_t>((l * field_rows + rin) * n + x);
            if (replayed) replayed[at] = v;
            if (intens) intens[at] = v.x * v.x + v.y * v.y;
        }
    }
}

#endif

template <class T>
__global__ void k_pad(const cx<T>* __restrict__ in, cx<T>* __restrict__ out, int w, int h, int pw, int ph, int C) {
    const size_t tot = static_cast<size_t>(pw) * ph * C;
    const int ox = (pw - w) / 2, oy = (ph - h) / 2;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < tot;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % pw);
        const int y = static_cast<int>((i / pw) % ph);
        const int c = static_cast<int>(i / (static_cast<size_t>(pw) * ph));
        const int sx = x - ox, sy = y - oy;
        out[i] = (sx >= 0 && sx < w && sy >= 0 && sy < h) ? in[(static_cast<size_t>(c) * h + sy) * w + sx]
                                                          : czero<T>();
    }
}

template <class T>
__global__ void k_crop(const cx<T>* __restrict__ in, cx<T>* __restrict__ out, int w, int h, int pw, int ph, int C) {
    const size_t tot = static_cast<size_t>(w) * h * C;
    const int ox = (pw - w) / 2, oy = (ph - h) / 2;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < tot;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % w);
        const int y = static_cast<int>((i / w) % h);
        const int c = static_cast<int>(i / (static_cast<size_t>(w) * h));
        out[i] = in[(static_cast<size_t>(c) * ph + y + oy) * pw + x + ox];
    }
}

template <class T>
__global__ void k_accumulate(const cx<T>* __restrict__ in, cx<T>* __restrict__ acc, size_t n, int first) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        acc[i] = first ? in[i] : acc[i] + in[i];
}

template <class T>
__global__ void k_intensity(const cx<T>* __restrict__ f, T* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const cx<T> v = f[i];
        if constexpr (sizeof(T) == 8)
            out[i] = __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));  // std::norm, uncontracted
        else
            out[i] = v.x * v.x + v.y * v.y;
    }
}

template <class T>
__global__ void k_tf(cx<T>* __restrict__ out, int w, int h, int C, const TfChan* __restrict__ tfc,
                     const double* __restrict__ fx, const double* __restrict__ fy) {
    const size_t tot = static_cast<size_t>(w) * h * C;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < tot;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % w);
        const int y = static_cast<int>((i / w) % h);
        const int c = static_cast<int>(i / (static_cast<size_t>(w) * h));
        out[i] = tf_value<T>(tfc[c], fx[x], fy[y]);
    }
}

// ------------------------------------------------------------------ host side

namespace {

constexpr int kThreads = 256;
constexpr size_t kSmemLimit = 227 * 1024;

template <class K>
void allow_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024) HC_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                        static_cast<int>(bytes)));
}

int grid_1d(holo_ctx* ctx, size_t n) {
    const size_t blocks = (n + kThreads - 1) / kThreads;
    const size_t cap = static_cast<size_t>(ctx->sm_count) * 8;
    return static_cast<int>(blocks < cap ? (blocks ? blocks : 1) : cap);
}

// rows per CTA for a row pass (ping-pong smem 2 * n * nb elements), targeting <= 64 KB
template <class T>
int rows_per_cta(int n) {
    const size_t per = 2 * static_cast<size_t>(n) * sizeof(cx<T>);
    if (per > kSmemLimit) throw Error(HOLO_ERR_CONFIG, "row length " + std::to_string(n) + " exceeds the on-chip FFT limit");
    int nb = static_cast<int>((64 * 1024) / per);
    if (nb < 1) nb = 1;
    if (nb > 16) nb = 16;
    return nb;
}

// columns per strip for a column pass with `buffers` smem buffers of h * nb elements
template <class T>
int cols_per_strip(int h, int buffers) {
    for (int nb : {8, 4, 2, 1})
        if (static_cast<size_t>(buffers) * h * nb * sizeof(cx<T>) <= 200 * 1024) return nb;
    throw Error(HOLO_ERR_CONFIG, "column length " + std::to_string(h) + " exceeds the on-chip FFT limit");
}

}  // namespace

template <class T>
void rows_fft(holo_ctx* ctx, const cx<T>* in, cx<T>* out, int n, long long nrows, int dir, T s) {
    if (nrows <= 0) return;
    const FftPlan plan = plan_or_throw(n);
    const int nb = rows_per_cta<T>(n);
    const size_t smem = 2 * static_cast<size_t>(n) * nb * sizeof(cx<T>);
    const long long grid = (nrows + nb - 1) / nb;
    const cx<T>* tw = ctx->twiddle<T>(n);
    if (dir < 0) {
        allow_smem(k_rows<T, -1>, smem);
        k_rows<T, -1><<<static_cast<unsigned>(grid), kThreads, smem, ctx->stream>>>(in, out, n, nrows, nb, plan, tw, s);
    } else {
        allow_smem(k_rows<T, +1>, smem);
        k_rows<T, +1><<<static_cast<unsigned>(grid), kThreads, smem, ctx->stream>>>(in, out, n, nrows, nb, plan, tw, s);
    }
    HC_LAUNCHED(ctx);
}

template <class T>
void cols_fft(holo_ctx* ctx, const cx<T>* in, cx<T>* out, int w, int h, int batch, int dir, T s) {
    if (batch <= 0) return;
    const FftPlan plan = plan_or_throw(h);
    const int nb = cols_per_strip<T>(h, 2);
    const size_t smem = 2 * static_cast<size_t>(h) * nb * sizeof(cx<T>);
    const dim3 grid((w + nb - 1) / nb, batch);
    const cx<T>* tw = ctx->twiddle<T>(h);
    if (dir < 0) {
        allow_smem(k_cols<T, -1>, smem);
        k_cols<T, -1><<<grid, kThreads, smem, ctx->stream>>>(in, out, w, h, nb, plan, tw, s);
    } else {
        allow_smem(k_cols<T, +1>, smem);
        k_cols<T, +1><<<grid, kThreads, smem, ctx->stream>>>(in, out, w, h, nb, plan, tw, s);
    }
    HC_LAUNCHED(ctx);
}

#ifdef HOLO_PROPAGATION_COMMON
// Fill the per-(plane, channel) constants for distances z[0..L) and wave channels.
std::vector<TfChan> make_tf_consts(const holo_wave& wave, const double* z, int L, int w, int h, int local_limit) {
    std::vector<TfChan> v(static_cast<size_t>(L) * wave.channels);
    const double two_pi = 2.0 * 3.141592653589793;
    for (int l = 0; l < L; ++l) {
        for (int c = 0; c < wave.channels; ++c) {
            const double lambda = wave.wavelengths[c];
            TfChan& p = v[static_cast<size_t>(l) * wave.channels + c];
            p.inv_l2 = 1.0 / (lambda * lambda);
            p.two_pi_z = two_pi * z[l];
            p.local = (local_limit && z[l] != 0.0) ? 1 : 0;
            p.fx_lim = p.fy_lim = 0.0;
            if (p.local) {
                // propagation.cpp:32-37
                const double du = 1.0 / (w * wave.pitch);
                const double dv = 1.0 / (h * wave.pitch);
                p.fx_lim = 1.0 / (lambda * std::sqrt((2.0 * du * z[l]) * (2.0 * du * z[l]) + 1.0));
                p.fy_lim = 1.0 / (lambda * std::sqrt((2.0 * dv * z[l]) * (2.0 * dv * z[l]) + 1.0));
            }
            const double inv_l = std::sqrt(p.inv_l2);
            p.inv_l = static_cast<float>(inv_l);
            p.two_pi_z_f = static_cast<float>(p.two_pi_z);
            // on-axis phase 2 pi z / lambda reduced into [0, 2 pi) in f64
            double ph = std::fmod(p.two_pi_z * inv_l, two_pi);
            if (ph < 0) ph += two_pi;
            p.phase0 = static_cast<float>(ph);
            const double dz2 = l + 1 < L ? two_pi * (z[l + 1] - z[l]) : 0.0;
            double dph = std::fmod(dz2 * inv_l, two_pi);
            if (dph < 0) dph += two_pi;
            p.step_phase = static_cast<float>(dph);
            p.step_2piz = static_cast<float>(dz2);
        }
    }
    return v;
}
#endif

template <class T>
void col_spectrum(holo_ctx* ctx, const cx<T>* layers, cx<T>* spec, int w, int h, int C, int L, const TfChan* d_tfc,
                  double pitch, const ColOpts<T>& opt) {
    const FftPlan plan = plan_or_throw(h);
    const int nb = cols_per_strip<T>(h, 3);
    const size_t smem = 3 * static_cast<size_t>(h) * nb * sizeof(cx<T>);
    allow_smem(k_col_spectrum<T>, smem);
    const dim3 grid((w + nb - 1) / nb, C);
    k_col_spectrum<T><<<grid, kThreads, smem, ctx->stream>>>(layers, spec, w, h, C, L, nb, plan, ctx->twiddle<T>(h),
                                                             d_tfc, ctx->freq(w, pitch), ctx->freq(h, pitch),
                                                             opt.tftab, opt.row_lo, opt.row_hi < 0 ? h : opt.row_hi);
    HC_LAUNCHED(ctx);
}

template <class T>
void col_replay(holo_ctx* ctx, const cx<T>* spec, cx<T>* out, int w, int h, int C, int nout, const int* d_plane_of,
                const TfChan* d_tfc, double pitch, const ColOpts<T>& opt) {
    if (nout <= 0) return;
    const FftPlan plan = plan_or_throw(h);
    const int nb = cols_per_strip<T>(h, 2);
    const size_t smem = 2 * static_cast<size_t>(h) * nb * sizeof(cx<T>);
    allow_smem(k_col_replay<T>, smem);
    const dim3 grid((w + nb - 1) / nb, C, nout);
    k_col_replay<T><<<grid, kThreads, smem, ctx->stream>>>(spec, out, w, h, C, nb, plan, ctx->twiddle<T>(h), d_tfc,
                                                           d_plane_of, ctx->freq(w, pitch), ctx->freq(h, pitch),
                                                           opt.tftab, opt.row_lo, opt.row_hi < 0 ? h : opt.row_hi);
    HC_LAUNCHED(ctx);
}

#ifdef HOLO_PROPAGATION_COMMON
void rows_epilogue(holo_ctx* ctx, const cx<float>* in, int w, int h, int C, int nout, int has_holo, cx<float>* holo,
                   cx<float>* replayed, float* intens) {
    const long long nrows = static_cast<long long>(nout) * C * h;
    if (nrows <= 0) return;
    const FftPlan plan = plan_or_throw(w);
    const int nb = rows_per_cta<float>(w);
    const size_t smem = 2 * static_cast<size_t>(w) * nb * sizeof(cx<float>);
    allow_smem(k_rows_epilogue, smem);
    const float s = static_cast<float>(1.0 / (static_cast<double>(w) * h));
    k_rows_epilogue<<<static_cast<unsigned>((nrows + nb - 1) / nb), kThreads, smem, ctx->stream>>>(
        in, w, nrows, nb, C, h, has_holo, plan, ctx->twiddle<float>(w), s, holo, replayed, intens);
    HC_LAUNCHED(ctx);
}
#endif

template <class T>
void pad_field(holo_ctx* ctx, const cx<T>* in, cx<T>* out, int w, int h, int C) {
    const size_t n = static_cast<size_t>(4) * w * h * C;
    k_pad<T><<<grid_1d(ctx, n), kThreads, 0, ctx->stream>>>(in, out, w, h, 2 * w, 2 * h, C);
    HC_LAUNCHED(ctx);
}

template <class T>
void crop_field(holo_ctx* ctx, const cx<T>* in, cx<T>* out, int w, int h, int C) {
    const size_t n = static_cast<size_t>(w) * h * C;
    k_crop<T><<<grid_1d(ctx, n), kThreads, 0, ctx->stream>>>(in, out, w, h, 2 * w, 2 * h, C);
    HC_LAUNCHED(ctx);
}

template <class T>
void accumulate(holo_ctx* ctx, const cx<T>* in, cx<T>* acc, size_t n, bool first) {
    k_accumulate<T><<<grid_1d(ctx, n), kThreads, 0, ctx->stream>>>(in, acc, n, first ? 1 : 0);
    HC_LAUNCHED(ctx);
}

template <class T>
void intensity(holo_ctx* ctx, const cx<T>* f, T* out, size_t n) {
    k_intensity<T><<<grid_1d(ctx, n), kThreads, 0, ctx->stream>>>(f, out, n);
    HC_LAUNCHED(ctx);
}

template <class T>
void transfer_function(holo_ctx* ctx, cx<T>* out, int w, int h, int C, const TfChan* d_tfc, double pitch) {
    const size_t n = static_cast<size_t>(w) * h * C;
    k_tf<T><<<grid_1d(ctx, n), kThreads, 0, ctx->stream>>>(out, w, h, C, d_tfc, ctx->freq(w, pitch),
                                                            ctx->freq(h, pitch));
    HC_LAUNCHED(ctx);
}

}  // namespace holo_cuda
