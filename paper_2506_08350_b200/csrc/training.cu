// The rest of a training step on the GPU (sm_100a): the loss terms of total_loss
// (proj/src/losses.cpp, ssim.cpp) with their gradient dL/dI, the opacity decay
// term (pipeline.cpp:47-52, 82-88) and the Adan / Adam update (optimizer.cpp).
//
// Precision and order: f64 throughout, like the reference, compiled without FMA
// contraction.  Sums that the reference folds row by row (fold_partials,
// common.hpp:70-74) are formed the same way -- each row summed along x in order
// (coalesced loads, transposed through shared memory), the rows then
// folded in order -- and the SSIM blurs are the reference's separable 11-tap
// correlations with zero extension (ssim.cpp:29-62) fused per 2-D tile, so on
// identical inputs the loss values and dL/dI equal the reference build's.  The
// opacity mean is a fixed-shape tree reduction (deterministic, not the
// reference's sequential order).
#include <cmath>
#include <vector>

#include "context.h"
#include "kernels.cuh"

namespace holo_cuda {

namespace {

constexpr int kWin = 11, kHalf = 5;
#ifndef HOLO_SSIM_TH
#define HOLO_SSIM_TH 16  // SSIM tile height: 16 measured best with gradients (32: +0.34 ms, 24: +0.09, 8: +0.68 at C3)
#endif
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

__constant__ double c_win[kWin];

// ---- row sums in the reference's order, coalesced
// One warp owns 32 rows.  Per 32-column chunk every lane loads its column of the
// 32 x 32 block (32 independent coalesced loads per array in flight), forms the
// per-element terms (and the elementwise gradient) there, and the block is
// transposed through shared memory so that lane r adds row r's 32 terms in x
// order -- the sequential fold of losses.cpp / ssim.cpp, so the row sums are the
// reference's bit for bit.
constexpr int kRowWarps = 2;

// loss_recon / loss_mse and the psnr rows (losses.cpp:28-132) over rows r of
// [L][C][H] (length W); grad = the pointwise term's gradient
template <bool PLAIN>
__global__ void __launch_bounds__(32 * kRowWarps) k_loss_row_sums(const double* __restrict__ I,
                                                                 const double* __restrict__ G,
                                                                 const double* __restrict__ masks, int C, int H,
                                                                 int W, long long nrows, double gscale,
                                                                 double* __restrict__ grad,
                                                                 double* __restrict__ rec_rows,
                                                                 double* __restrict__ mse_rows) {
    __shared__ double tile[kRowWarps][PLAIN ? 1 : 2][32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long r0 = (static_cast<long long>(blockIdx.x) * kRowWarps + warp) * 32;
    if (r0 >= nrows) return;
    const int nr = static_cast<int>(min(32LL, nrows - r0));
    // per-row offsets, computed once by lane j for row r0 + j and broadcast
    const long long myrow = r0 + min(lane, nr - 1);
    const long long moff_l = PLAIN ? 0 : (myrow / (static_cast<long long>(C) * H) * H + myrow % H) * W;
    double acc0 = 0.0, acc1 = 0.0;
    for (int c0 = 0; c0 < W; c0 += 32) {
        const int nc = min(32, W - c0);
        // every lane loads (the tail lanes repeat the last column) so that the row
        // offsets can be broadcast with full-warp shuffles
        const bool live = lane < nc;
        const int x = c0 + (live ? lane : nc - 1);
        double a[32], b[32], m[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (j < nr) {
                const size_t i = static_cast<size_t>(r0 + j) * W + x;
                a[j] = I[i];
                b[j] = G[i];
                if (!PLAIN) m[j] = masks[__shfl_sync(0xffffffffu, moff_l, j) + x];
            }
        }
        if (live) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (j < nr) {
                    const size_t i = static_cast<size_t>(r0 + j) * W + x;
                    const double e = a[j] - b[j];
                    if (PLAIN) {
                        tile[warp][0][j][lane] = e * e;
                        if (grad) grad[i] = gscale * e;
                    } else {
                        const double weight = 1.0 + m[j] * m[j] + b[j] * b[j];
                        tile[warp][0][j][lane] = weight * e * e;
                        tile[warp][PLAIN ? 0 : 1][j][lane] = e * e;
                        if (grad) grad[i] = gscale * weight * e;
                    }
                }
            }
        }
        __syncwarp();
        if (lane < nr) {
            for (int k = 0; k < nc; ++k) {
                acc0 += tile[warp][0][lane][k];
                if (!PLAIN) acc1 += tile[warp][PLAIN ? 0 : 1][lane][k];
            }
        }
        __syncwarp();
    }
    if (lane < nr) {
        rec_rows[r0 + lane] = acc0;
        mse_rows[r0 + lane] = PLAIN ? acc0 : acc1;
    }
}

// SSIM map row sums over the valid window centres (ssim.cpp:100-121): rows r of
// [L][C][vrows], columns [5, W - 5)
__global__ void __launch_bounds__(32 * kRowWarps) k_ssim_row_sums(const double* __restrict__ smap, int W, int H,
                                                                 int vrows, long long nrows,
                                                                 double* __restrict__ out) {
    __shared__ double tile[kRowWarps][32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long r0 = (static_cast<long long>(blockIdx.x) * kRowWarps + warp) * 32;
    if (r0 >= nrows) return;
    const int nr = static_cast<int>(min(32LL, nrows - r0));
    const long long myrow = r0 + min(lane, nr - 1);
    const long long off_l = myrow / vrows * static_cast<long long>(W) * H + (myrow % vrows + 5) * W + 5;
    const int ncols = W - 10;
    double acc = 0.0;
    for (int c0 = 0; c0 < ncols; c0 += 32) {
        const int nc = min(32, ncols - c0);
        const int x = c0 + min(lane, nc - 1);  // all lanes load: full-warp shuffles
        double v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nr) v[j] = smap[__shfl_sync(0xffffffffu, off_l, j) + x];
        if (lane < nc) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j < nr) tile[warp][j][lane] = v[j];
        }
        __syncwarp();
        if (lane < nr)
            for (int k = 0; k < nc; ++k) acc += tile[warp][lane][k];
        __syncwarp();
    }
    if (lane < nr) out[r0 + lane] = acc;
}

// out[t] = mul * (sum of v[t * len .. t * len + len) in order) / div, one warp per
// segment: the warp stages 256-value chunks in shared memory (coalesced) and lane 0
// adds them in order -- loads run ahead, only the f64 add chain is serial.  Two
// independent jobs (v0 / v1) can share a launch: warps t >= nseg take the second.
struct FoldJob {
    const double* v;
    double mul, div;
    double* out;
};
constexpr int kFoldChunk = 256;
__global__ void __launch_bounds__(128) k_fold_seg(FoldJob j0, FoldJob j1, int nseg, int len) {
    __shared__ double buf[4][kFoldChunk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int t = blockIdx.x * 4 + warp;
    if (t >= 2 * nseg || (t >= nseg && j1.v == nullptr)) return;
    const FoldJob& job = t < nseg ? j0 : j1;
    if (t >= nseg) t -= nseg;
    const double* p = job.v + static_cast<size_t>(t) * len;
    double* sb = buf[warp];
    double acc = 0.0;
    for (int c0 = 0; c0 < len; c0 += kFoldChunk) {
        const int nc = min(kFoldChunk, len - c0);
        for (int k = lane; k < nc; k += 32) sb[k] = p[c0 + k];
        __syncwarp();
        if (lane == 0) {
#pragma unroll 16
            for (int k = 0; k < nc; ++k) acc += sb[k];
        }
        __syncwarp();
    }
    if (lane == 0) job.out[t] = job.mul * acc / job.div;
}

void fold(holo_ctx* ctx, int nseg, int len, const FoldJob& a, const FoldJob& b = FoldJob{nullptr, 1.0, 1.0, nullptr}) {
    const int warps = b.v ? 2 * nseg : nseg;
    k_fold_seg<<<(warps + 3) / 4, 128, 0, ctx->stream>>>(a, b, nseg, len);
    HC_LAUNCHED(ctx);
}

__global__ void k_fill(double* p, int n, double v) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = v;
}

// ---- SSIM (ssim.cpp:64-147), fused per 2-D tile
// Forward: the tile's I and I_gt with a 5-pixel halo (zeros outside the image:
// the zero extension of corr_h / corr_v adds exact zeros) go to shared memory;
// the horizontal 11-tap pass forms mx, my, qx, qy, qxy for the tile's rows plus
// the halo rows, the vertical pass finishes them per pixel, and the SSIM value and
// the three gradient maps (zero outside the valid window centres) are written.
// Backward: the same two passes over the gradient maps, then
// grad -= scale (inv_n (t1 + 2 x t2 + y t3)).  Each tap sum runs k = 0..10 in
// order with separate multiply and add, as the reference's loops.
constexpr int kTW = 32, kTH = HOLO_SSIM_TH, kHW = kTW + 2 * kHalf, kHH = kTH + 2 * kHalf;
constexpr size_t kSsimFwdSmem = sizeof(double) * (2 * kHH * kHW + 5 * kHH * kTW);
constexpr size_t kSsimBwdSmem = sizeof(double) * (3 * kHH * kHW + 3 * kHH * kTW);

template <int Q>
__device__ __forceinline__ void load_halo(const double* const* src, size_t base, int W, int H, int x0, int y0,
                                          double* dst) {
    for (int i = threadIdx.x; i < kHH * kHW; i += blockDim.x) {
        const int r = i / kHW, c = i % kHW;
        const int gy = y0 - kHalf + r, gx = x0 - kHalf + c;
        const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
        const size_t gi = base + static_cast<size_t>(gy) * W + gx;
#pragma unroll
        for (int q = 0; q < Q; ++q) dst[q * kHH * kHW + i] = in ? src[q][gi] : 0.0;
    }
}

// The horizontal pass gives each thread two adjacent outputs of a row (the 12
// inputs they share are read once, as 16-byte pairs); the vertical pass gives
// each thread four consecutive rows of a column (14 inputs per quantity for four
// outputs).  Each output's 11-tap sum still runs k = 0..10 in order.
constexpr int kHP = 2, kVP = kTH / 8;  // outputs per thread in the horizontal / vertical pass
static_assert(kTH % kVP == 0 && kTW * (kTH / kVP) == 256, "one vertical item per thread");
static_assert(kHW % 2 == 0 && (kHH * kHW) % 2 == 0 && kTW % kHP == 0, "16-byte aligned row pairs");

// 12 consecutive values starting at an even (16-byte aligned) index
__device__ __forceinline__ void load12(const double* p, double (&v)[12]) {
    const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const double2 t = q[k];
        v[2 * k] = t.x;
        v[2 * k + 1] = t.y;
    }
}

// out[o] = sum_k w[k] val[o + k], k = 0..10, for o < kHP
__device__ __forceinline__ void tap2(const double (&val)[12], double (&out)[kHP]) {
#pragma unroll
    for (int o = 0; o < kHP; ++o) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < kWin; ++k) acc += c_win[k] * val[o + k];
        out[o] = acc;
    }
}

// vertical: out[o] = sum_k w[k] col[(o + k) * kTW], o < kVP
__device__ __forceinline__ void tap_v(const double* col, double (&out)[kVP]) {
    double v[kVP + kWin - 1];
#pragma unroll
    for (int k = 0; k < kVP + kWin - 1; ++k) v[k] = col[k * kTW];
#pragma unroll
    for (int o = 0; o < kVP; ++o) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < kWin; ++k) acc += c_win[k] * v[o + k];
        out[o] = acc;
    }
}

template <bool GRAD>
__global__ void __launch_bounds__(256) k_ssim_fwd(const double* __restrict__ X, const double* __restrict__ Y, int W,
                                                  int H, double* __restrict__ smap, double* __restrict__ gmaps,
                                                  size_t gstride) {
    extern __shared__ __align__(16) double sm[];
    double* sxy = sm;                 // [2][kHH][kHW]
    double* hb = sm + 2 * kHH * kHW;  // [5][kHH][kTW]
    const size_t P = static_cast<size_t>(W) * H;
    const size_t base = blockIdx.z * P;
    const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
    const double* src[2] = {X, Y};
    load_halo<2>(src, base, W, H, x0, y0, sxy);
    __syncthreads();
    for (int it = threadIdx.x; it < kHH * (kTW / kHP); it += blockDim.x) {
        const int r = it / (kTW / kHP), c = kHP * (it % (kTW / kHP));
        double xv[12], yv[12], val[12], o[kHP];
        load12(sxy + r * kHW + c, xv);
        load12(sxy + kHH * kHW + r * kHW + c, yv);
        double* dst = hb + r * kTW + c;
        tap2(xv, o);  // mx
#pragma unroll
        for (int e = 0; e < kHP; ++e) dst[e] = o[e];
        tap2(yv, o);  // my
#pragma unroll
        for (int e = 0; e < kHP; ++e) dst[kHH * kTW + e] = o[e];
#pragma unroll
        for (int k = 0; k < 12; ++k) val[k] = xv[k] * xv[k];
        tap2(val, o);  // qx
#pragma unroll
        for (int e = 0; e < kHP; ++e) dst[2 * kHH * kTW + e] = o[e];
#pragma unroll
        for (int k = 0; k < 12; ++k) val[k] = yv[k] * yv[k];
        tap2(val, o);  // qy
#pragma unroll
        for (int e = 0; e < kHP; ++e) dst[3 * kHH * kTW + e] = o[e];
#pragma unroll
        for (int k = 0; k < 12; ++k) val[k] = xv[k] * yv[k];
        tap2(val, o);  // qxy
#pragma unroll
        for (int e = 0; e < kHP; ++e) dst[4 * kHH * kTW + e] = o[e];
    }
    __syncthreads();
    {
        const int c = threadIdx.x % kTW, r0 = kVP * (threadIdx.x / kTW);
        double m[5][kVP];
#pragma unroll
        for (int q = 0; q < 5; ++q) tap_v(hb + q * kHH * kTW + r0 * kTW + c, m[q]);
#pragma unroll
        for (int o = 0; o < kVP; ++o) {
            const int py = y0 + r0 + o, px = x0 + c;
            if (py >= H || px >= W) continue;
            const bool valid = px >= kHalf && px < W - kHalf && py >= kHalf && py < H - kHalf;
            double s = 0.0, gmu = 0.0, gqx = 0.0, gqxy = 0.0;
            if (valid) {
                const double ux = m[0][o], uy = m[1][o];
                const double vxv = m[2][o] - ux * ux;
                const double vyv = m[3][o] - uy * uy;
                const double vxy = m[4][o] - ux * uy;
                const double a1 = 2.0 * ux * uy + kC1;
                const double a2 = 2.0 * vxy + kC2;
                const double b1 = ux * ux + uy * uy + kC1;
                const double b2 = vxv + vyv + kC2;
                const double d = b1 * b2;
                s = (a1 * a2) / d;
                if (GRAD) {
                    gmu = (2.0 * uy * (a2 - a1) - s * 2.0 * ux * (b2 - b1)) / d;
                    gqx = -s / b2;
                    gqxy = 2.0 * a1 / d;
                }
            }
            const size_t gi = base + static_cast<size_t>(py) * W + px;
            smap[gi] = s;
            if (GRAD) {
                const size_t li = blockIdx.z * P + static_cast<size_t>(py) * W + px;
                gmaps[li] = gmu;
                gmaps[gstride + li] = gqx;
                gmaps[2 * gstride + li] = gqxy;
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_ssim_bwd(const double* __restrict__ gmaps, size_t gstride,
                                                  const double* __restrict__ X, const double* __restrict__ Y, int W,
                                                  int H, double inv_n, double scale, double* __restrict__ grad) {
    extern __shared__ __align__(16) double sm[];
    double* sg = sm;                  // [3][kHH][kHW]
    double* hb = sm + 3 * kHH * kHW;  // [3][kHH][kTW]
    const size_t P = static_cast<size_t>(W) * H;
    const size_t lbase = blockIdx.z * P;
    const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
    const double* src[3] = {gmaps, gmaps + gstride, gmaps + 2 * gstride};
    load_halo<3>(src, lbase, W, H, x0, y0, sg);
    __syncthreads();
    for (int it = threadIdx.x; it < kHH * (kTW / kHP); it += blockDim.x) {
        const int r = it / (kTW / kHP), c = kHP * (it % (kTW / kHP));
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            double v[12], o[kHP];
            load12(sg + q * kHH * kHW + r * kHW + c, v);
            tap2(v, o);
#pragma unroll
            for (int e = 0; e < kHP; ++e) hb[q * kHH * kTW + r * kTW + c + e] = o[e];
        }
    }
    __syncthreads();
    const int c = threadIdx.x % kTW, r0 = kVP * (threadIdx.x / kTW);
    double t[3][kVP];
#pragma unroll
    for (int q = 0; q < 3; ++q) tap_v(hb + q * kHH * kTW + r0 * kTW + c, t[q]);
#pragma unroll
    for (int o = 0; o < kVP; ++o) {
        const int py = y0 + r0 + o, px = x0 + c;
        if (py >= H || px >= W) continue;
        const size_t gi = lbase + static_cast<size_t>(py) * W + px;
        grad[gi] -= scale * (inv_n * (t[0][o] + 2.0 * X[gi] * t[1][o] + Y[gi] * t[2][o]));
    }
}

__global__ void k_f32_to_f64(const float* __restrict__ in, double* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<double>(in[i]);
}

// |v|^2 in f64 of the fp32 replay, rounded like intensity() of the widened field
__global__ void k_replay_intensity(const cx<float>* __restrict__ rep, double* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double x = rep[i].x, y = rep[i].y;
        out[i] = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    }
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
// (masks [L][H][W]); grad (optional) is overwritten with dL/dI.
// d_out[0] = recon, d_out[1 + l] = mean SSIM of plane l, d_out[1 + L + l] =
// the mse of plane l; the host finishes the scalar algebra.
void ssim_setup() {
    // per device: constant memory and function attributes belong to a device
    static bool done[256] = {};
    int dev = 0;
    HC_CUDA(cudaGetDevice(&dev));
    bool& win_set = done[dev & 255];
    if (!win_set) {  // ssim.cpp:16-26
        double w[kWin], sum = 0.0;
        for (int i = 0; i < kWin; ++i) {
            const double d = i - kHalf;
            w[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            sum += w[i];
        }
        for (double& v : w) v /= sum;
        HC_CUDA(cudaMemcpyToSymbol(c_win, w, sizeof w));
        HC_CUDA(cudaFuncSetAttribute(k_ssim_fwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kSsimFwdSmem)));
        HC_CUDA(cudaFuncSetAttribute(k_ssim_fwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kSsimFwdSmem)));
        HC_CUDA(cudaFuncSetAttribute(k_ssim_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kSsimBwdSmem)));
        win_set = true;
    }
}

void losses_gpu(holo_ctx* ctx, const double* I, const double* G, const double* masks, int L, int C, int H, int W,
                bool plain, bool with_ssim, double lambda_ssim, double* grad, double* d_out) {
    const size_t n = static_cast<size_t>(C) * H * W;
    if (with_ssim && (W < kWin || H < kWin))
        throw Error(HOLO_ERR_CONFIG, "ssim needs images at least 11 pixels in each dimension");
    ssim_setup();
    const long long rows_n = static_cast<long long>(L) * C * H;
    double* rows = static_cast<double*>(ctx->buffer("loss_rows", sizeof(double) * 2 * rows_n));
    double* prow = rows + rows_n;
    double* lsum = static_cast<double*>(ctx->buffer("loss_plane", sizeof(double) * L));
    const double inv_l = 1.0 / static_cast<double>(L), inv_n = 1.0 / static_cast<double>(n);
    // recon / mse and the psnr rows in one pass (losses.cpp:28-132); grad = the
    // pointwise term's gradient (the reference adds it to a zeroed stack)
    const unsigned rb = static_cast<unsigned>((rows_n + 32 * kRowWarps - 1) / (32 * kRowWarps));
    const double gscale = 2.0 * inv_l * inv_n;
    if (plain)
        k_loss_row_sums<true><<<rb, 32 * kRowWarps, 0, ctx->stream>>>(I, G, masks, C, H, W, rows_n, gscale, grad,
                                                                      rows, prow);
    else
        k_loss_row_sums<false><<<rb, 32 * kRowWarps, 0, ctx->stream>>>(I, G, masks, C, H, W, rows_n, gscale, grad,
                                                                       rows, prow);
    HC_LAUNCHED(ctx);
    // per plane: the recon rows (times inv_l inv_n) and the psnr rows (over n), one launch
    fold(ctx, L, C * H, FoldJob{rows, inv_l * inv_n, 1.0, lsum}, FoldJob{prow, 1.0, static_cast<double>(n), d_out + 1 + L});
    fold(ctx, 1, L, FoldJob{lsum, 1.0, 1.0, d_out});

    if (!with_ssim) {  // the SSIM term left out: mean SSIM 1 contributes 0
        k_fill<<<1, 32, 0, ctx->stream>>>(d_out + 1, L, 1.0);
        HC_LAUNCHED(ctx);
        return;
    }
    ssim_gpu(ctx, I, G, L, C, H, W, lambda_ssim / static_cast<double>(L), grad, d_out + 1);
}

// mean SSIM per plane (ssim_mean, ssim.cpp:64-147) of stacks [L][C][H][W] into
// d_mean[L]; with grad, grad -= gscale * d(mean SSIM_l)/dI_l (loss_ssim's
// accumulation, losses.cpp:104-108)
void ssim_gpu(holo_ctx* ctx, const double* I, const double* G, int L, int C, int H, int W, double gscale,
              double* grad, double* d_mean) {
    if (W < kWin || H < kWin) throw Error(HOLO_ERR_CONFIG, "ssim needs images at least 11 pixels in each dimension");
    ssim_setup();
    const size_t n = static_cast<size_t>(C) * H * W;
    const int vrows = H - 2 * kHalf;
    const size_t n_valid = static_cast<size_t>(W - 2 * kHalf) * vrows * C;
    double* smap = static_cast<double*>(ctx->buffer("ssim_map", sizeof(double) * L * n));
    double* gmaps = grad ? static_cast<double*>(ctx->buffer("ssim_gmaps", sizeof(double) * 3 * n)) : nullptr;
    const dim3 tg((W + kTW - 1) / kTW, (H + kTH - 1) / kTH, C);
    for (int l = 0; l < L; ++l) {
        const size_t off = static_cast<size_t>(l) * n;
        if (grad) {
            k_ssim_fwd<true><<<tg, 256, kSsimFwdSmem, ctx->stream>>>(I + off, G + off, W, H, smap + off, gmaps, n);
            HC_LAUNCHED(ctx);
            k_ssim_bwd<<<tg, 256, kSsimBwdSmem, ctx->stream>>>(gmaps, n, I + off, G + off, W, H,
                                                              1.0 / static_cast<double>(n_valid),
                                                              gscale, grad + off);
            HC_LAUNCHED(ctx);
        } else {
            k_ssim_fwd<false><<<tg, 256, kSsimFwdSmem, ctx->stream>>>(I + off, G + off, W, H, smap + off, nullptr, 0);
            HC_LAUNCHED(ctx);
        }
    }
    const long long srows_n = static_cast<long long>(L) * C * vrows;
    double* srows = static_cast<double*>(ctx->buffer("ssim_rows", sizeof(double) * srows_n));
    double* ssum = static_cast<double*>(ctx->buffer("ssim_sum", sizeof(double) * L * C));
    k_ssim_row_sums<<<static_cast<unsigned>((srows_n + 32 * kRowWarps - 1) / (32 * kRowWarps)), 32 * kRowWarps, 0,
                      ctx->stream>>>(smap, W, H, vrows, srows_n, srows);
    HC_LAUNCHED(ctx);
    // per (plane, channel) the rows in order; per plane the channels in order, / n_valid
    fold(ctx, L * C, vrows, FoldJob{srows, 1.0, 1.0, ssum});
    fold(ctx, L, C, FoldJob{ssum, 1.0, static_cast<double>(n_valid), d_mean});
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

void replay_intensity_f64(holo_ctx* ctx, const cx<float>* rep, double* out, size_t n) {
    k_replay_intensity<<<blocks_for(n), 256, 0, ctx->stream>>>(rep, out, n);
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
