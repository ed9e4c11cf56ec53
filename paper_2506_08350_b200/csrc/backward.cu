// Backward of the render (sm_100a): raster_backward (proj/src/rasterizer.cpp:332-528)
// and the seed of the adjoint propagation chain of total_loss (pipeline.cpp:63-80).
//
//   k_bwd_seed      gv_l = 2 replayed_l . dL/dI_l                  (pipeline.cpp:68-70)
//   (adjoint propagation = the forward recording + replay applied to gv, capi.cu)
//   k_bwd_prep      per Gaussian: cos / sin of the phases, amplitudes (fp32)
//   k_raster_bwd    one CTA per (plane, tile) bucket, one thread per pixel:
//                   replay the forward to find the pixel's accepted entries
//                   (the same staged records and instruction sequence as
//                   k_composite, raster_eval.cuh), then the back-to-front sweep
//                   recovering T and the colour behind (rasterizer.cpp:376-428);
//                   per-entry gradients are reduced over the warp, then over
//                   the CTA's warps in warp order (deterministic) into egrad[entry][13]
//   k_bwd_gauss     per Gaussian, f64: sums its entries' gradients in entry
//                   (bucket) order, the reference's merge order (:435-455), then
//                   the chain to the stored parameters (:458-525) with
//                   covariance_backward (scene.cpp:84-121) and the straight-through
//                   plane-logit route (ste_assign, scene.cpp:132-152)
#include "raster_eval.cuh"

namespace holo_cuda {

namespace {

// per-entry gradient slots (EntryGrad, rasterizer.cpp:321-328)
enum { kGMuX = 0, kGMuY, kGI00, kGI01, kGI11, kGAlpha, kGRho, kGAmp, kGPh = kGAmp + 3, kGradVals = kGPh + 3 };

constexpr float kInvScale = -1.38629436111989061883f;  // 1 / (GRec conic scale -log2(e) / 2) = -2 ln 2

// dL/dI as float, or as double (total_loss's f64 loss gradient, narrowed here)
template <class G>
__global__ void k_bwd_seed(const cx<float>* __restrict__ rep, const G* __restrict__ gi, cx<float>* __restrict__ gv,
                           size_t n) {
    for (size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; t < n;
         t += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const float s = 2.0f * static_cast<float>(gi[t]);
        gv[t] = scale(rep[t], s);
    }
}

__global__ void k_bwd_prep(const double* __restrict__ amplitudes, const double* __restrict__ phases,
                           const GRec* __restrict__ rec, size_t N, BwdRec* __restrict__ out) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= N) return;
    BwdRec r;
    for (int c = 0; c < 3; ++c) {
        double s, co;
        sincos(phases[3 * i + c], &s, &co);
        r.cs[2 * c] = static_cast<float>(co);
        r.cs[2 * c + 1] = static_cast<float>(s);
        r.amp[c] = static_cast<float>(amplitudes[3 * i + c]);
    }
    r.alpha = rec[i].alpha;
    r.pad[0] = r.pad[1] = 0.0f;
    out[i] = r;
}

// One step of a warp reduce-scatter over 2H values: lanes with bit D set keep
// (and receive the partner's copy of) the upper half, the others the lower half.
template <int D, int H>
__device__ __forceinline__ void reduce_scatter_step(float (&w)[16], int lane) {
    const bool up = (lane & D) != 0;
#pragma unroll
    for (int i = 0; i < H; ++i) {
        const float send = up ? w[i] : w[i + H];
        const float keep = up ? w[i + H] : w[i];
        w[i] = keep + __shfl_xor_sync(0xffffffffu, send, D);
    }
}

template <int TILE, int C>
__global__ void __launch_bounds__(TILE * TILE) k_raster_bwd(RasterBwdArgs a) {
    constexpr int NT = TILE * TILE;
    constexpr int kStage = TILE == 32 ? 32 : 128;  // entries per batch (per-warp partials: 53 KB at 16x16)
    constexpr int kBlocksX = TILE / 8;
    __shared__ Staged s_rec[kStage];
    __shared__ float4 s_box[kStage];
    __shared__ int s_g[kStage];
    __shared__ BwdRec s_brec[kStage];  // pad[0] carries rho
    __shared__ float s_acc[kStage * kGradVals];
    // per-warp partials of the batch's entries, summed over the warps in a fixed
    // order once per batch (deterministic: no float atomics, one barrier pair per
    // batch rather than per 32-entry chunk)
    extern __shared__ float s_part[];  // [NT / 32][kStage][kGradVals]
    constexpr int NW = NT / 32;

    const int tx = blockIdx.x, ty = blockIdx.y, lplane = blockIdx.z;
    const int lb = (lplane * gridDim.y + ty) * gridDim.x + tx;
    const int px0 = tx * TILE, py0 = ty * TILE;
    const unsigned e0 = min(a.bstart[lb], a.capacity);
    const int n = static_cast<int>(min(a.bstart[lb + 1], a.capacity) - e0);
    if (n == 0) return;  // CTA-uniform
    const int plane = a.plane_begin + lplane;

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int bx = (warp % kBlocksX) * 8, by = (warp / kBlocksX) * 4;
    const int lx = bx + (lane & 7), ly = by + (lane >> 3);
    const int px = px0 + lx, py = py0 + ly;
    const bool inside = px < a.W && py < a.H;
    const float fx = static_cast<float>(lx) + 0.5f, fy = static_cast<float>(ly) + 0.5f;
    const float bxlo = static_cast<float>(bx) + 0.5f, bxhi = static_cast<float>(bx) + 7.5f;
    const float bylo = static_cast<float>(by) + 0.5f, byhi = static_cast<float>(by) + 3.5f;
    const float thr = a.floor_positive ? a.alpha_floor : 0.0f;
    const float clamp = a.alpha_clamp;
    const size_t P = static_cast<size_t>(a.W) * a.H;
    const size_t pix = static_cast<size_t>(py) * a.W + px;

    // upstream gradient of this pixel, and the forward's outcome there
    cx<float> g[C];
    int contrib = 0;
    bool any = false;
    float T = 1.0f;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        g[c] = inside ? a.grad_layers[(static_cast<size_t>(lplane) * C + c) * P + pix] : mk(0.0f, 0.0f);
        any = any || g[c].x != 0.0f || g[c].y != 0.0f;
    }
    if (inside) {
        contrib = a.n_contrib[static_cast<size_t>(lplane) * P + pix];
        T = a.t_final[static_cast<size_t>(lplane) * P + pix];
    }
    const bool active = inside && contrib > 0 && any;

    auto stage = [&](int base, int cnt) {
        for (int t = tid; t < cnt; t += NT) {
            const int gi = a.egidx[e0 + base + t];
            const GRec r = a.rec[gi];
            float alpha = r.alpha, rho = 1.0f;
            if (a.soft) {
                rho = static_cast<float>(a.rho[static_cast<size_t>(gi) * a.L + plane]);
                alpha = static_cast<float>(static_cast<double>(r.alpha) * a.rho[static_cast<size_t>(gi) * a.L + plane]);
            }
            stage_entry(r, px0, py0, alpha, s_rec[t], s_box[t]);
            BwdRec br = a.brec[gi];
            br.pad[0] = rho;
            s_brec[t] = br;
            s_g[t] = gi;
        }
    };

    // ---- pass 1: the forward's accepted set -- the first n_contrib accepted
    // entries in bucket order (rasterizer.cpp:379-387)
    int k = 0, e_last = -1;
    const bool replay = a.e_last == nullptr;  // else the forward recorded e_last
    if (!replay && inside) e_last = a.e_last[static_cast<size_t>(lplane) * P + pix];
    for (int base = 0; replay && base < n; base += kStage) {
        const int cnt = min(n - base, kStage);
        stage(base, cnt);
        __syncthreads();
        for (int c0 = 0; c0 < cnt; c0 += 32) {
            const bool searching = active && k < contrib;
            if (!__any_sync(0xffffffffu, searching)) break;
            const bool hit = c0 + lane < cnt && box_hits(s_box[c0 + lane], bxlo, bxhi, bylo, byhi);
            unsigned mask = __ballot_sync(0xffffffffu, hit);
            while (mask) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                float4 B;
                const float al = eval_alpha(&s_rec[c0 + j], fx, fy, clamp, B);
                if (active && k < contrib && al > thr) {
                    ++k;
                    if (k == contrib) e_last = base + c0 + j;
                }
            }
        }
        __syncthreads();
    }

    // ---- pass 2: back to front from e_last (rasterizer.cpp:389-428)
    cx<float> accum[C], last[C];
#pragma unroll
    for (int c = 0; c < C; ++c) accum[c] = last[c] = mk(0.0f, 0.0f);
    float last_alpha = 0.0f;
    const int nb = (n + kStage - 1) / kStage;
    for (int bi = nb - 1; bi >= 0; --bi) {
        const int base = bi * kStage;
        const int cnt = min(n - base, kStage);
        if (nb > 1 || !replay) stage(base, cnt);  // one batch: still staged from pass 1
        __syncthreads();
        float* my_part = s_part + warp * kStage * kGradVals;
        for (int i = lane; i < cnt * kGradVals; i += 32) my_part[i] = 0.0f;
        __syncwarp();
        for (int c0 = ((cnt - 1) / 32) * 32; c0 >= 0; c0 -= 32) {
            const bool live = active && e_last >= base + c0;
            if (__any_sync(0xffffffffu, live)) {
                const bool hit = c0 + lane < cnt && box_hits(s_box[c0 + lane], bxlo, bxhi, bylo, byhi);
                unsigned mask = __ballot_sync(0xffffffffu, hit);
                while (mask) {
                    const int j = 31 - __clz(mask);  // highest first
                    mask &= ~(1u << j);
                    const int er = base + c0 + j;
                    const Staged* e = &s_rec[c0 + j];
                    float4 B;
                    const float al = eval_alpha(e, fx, fy, clamp, B);
                    const bool acc = active && er <= e_last && al > thr;
                    if (!__any_sync(0xffffffffu, acc)) continue;
                    float v[kGradVals];
#pragma unroll
                    for (int q = 0; q < kGradVals; ++q) v[q] = 0.0f;
                    if (acc) {
                        const BwdRec& br = s_brec[c0 + j];
                        T = __fdividef(T, 1.0f - al);
                        const float aw = al * T;
                        float d_alpha = 0.0f;
                        const float4 Cc = e->c;
#pragma unroll
                        for (int c = 0; c < C; ++c) {
                            const cx<float> vc = c == 0 ? mk(B.z, B.w) : (c == 1 ? mk(Cc.x, Cc.y) : mk(Cc.z, Cc.w));
                            accum[c] = mk(last_alpha * last[c].x + (1.0f - last_alpha) * accum[c].x,
                                          last_alpha * last[c].y + (1.0f - last_alpha) * accum[c].y);
                            last[c] = vc;
                            d_alpha += (vc.x - accum[c].x) * g[c].x + (vc.y - accum[c].y) * g[c].y;
                            const float co = br.cs[2 * c], si = br.cs[2 * c + 1];
                            v[kGAmp + c] = aw * (co * g[c].x + si * g[c].y);
                            v[kGPh + c] = aw * br.amp[c] * (-si * g[c].x + co * g[c].y);
                        }
                        last_alpha = al;
                        d_alpha *= T;
                        if (al < clamp) {
                            // alpha_eff = alpha_sig * gauss * rho below the clamp
                            const float4 A = e->a;
                            const float dx = fx - A.x, dy = fy - A.y;
                            const float t = fmaf(A.w, dy, A.z * dx);
                            const float gauss = ex2_approx(fmaf(B.x * dy, dy, dx * t));
                            const float alpha_sig = br.alpha;
                            const float rho = br.pad[0];
                            v[kGAlpha] = d_alpha * gauss * rho;
                            v[kGRho] = d_alpha * alpha_sig * gauss;
                            const float gg = d_alpha * alpha_sig * rho * gauss;
                            const float i00 = A.z * kInvScale, i01 = A.w * (0.5f * kInvScale), i11 = B.x * kInvScale;
                            v[kGMuX] = gg * (i00 * dx + i01 * dy);
                            v[kGMuY] = gg * (i01 * dx + i11 * dy);
                            v[kGI00] = gg * (-0.5f * dx * dx);
                            v[kGI01] = gg * (-dx * dy);
                            v[kGI11] = gg * (-0.5f * dy * dy);
                        }
                    }
                    // reduce-scatter over the warp: afterwards lanes 2q, 2q+1 hold the
                    // warp's sum of value q (16 shuffles instead of 13 x 5)
                    float w[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) w[q] = q < kGradVals ? v[q] : 0.0f;
                    reduce_scatter_step<16, 8>(w, lane);
                    reduce_scatter_step<8, 4>(w, lane);
                    reduce_scatter_step<4, 2>(w, lane);
                    reduce_scatter_step<2, 1>(w, lane);
                    w[0] += __shfl_xor_sync(0xffffffffu, w[0], 1);
                    const int q = (lane >> 1) & 15;
                    if ((lane & 1) == 0 && q < kGradVals) my_part[(c0 + j) * kGradVals + q] = w[0];
                }
            }
        }
        __syncthreads();
        // the batch's entries: warp partials summed in warp order
        for (int i = tid; i < cnt * kGradVals; i += NT) {
            float sum = 0.0f;
#pragma unroll
            for (int wi = 0; wi < NW; ++wi) sum += s_part[wi * kStage * kGradVals + i];
            s_acc[i] = sum;
        }
        __syncthreads();
        // egrad is ordered per Gaussian: its k-th entry (bucket order: plane, then
        // tile row, then tile column) at goff[g] + k, so the merge reads it in the
        // reference's order without searching the buckets
        for (int t = tid; t < cnt; t += NT) {
            const int gi = s_g[t];
            const int4 r = a.rect[gi];
            const int area = (r.y - r.x) * (r.w - r.z);
            int k = (ty - r.z) * (r.y - r.x) + (tx - r.x);
            if (a.soft) k += __popcll(a.pmask[gi] & ((1ull << plane) - 1ull)) * area;
            float* dst = a.egrad + (static_cast<size_t>(a.goff[gi]) + k) * kGradVals;
#pragma unroll
            for (int q = 0; q < kGradVals; ++q) dst[q] = s_acc[t * kGradVals + q];
        }
        __syncthreads();
    }
}

// ---- per-Gaussian chain (f64)

__global__ void __launch_bounds__(256) k_bwd_gauss(GaussBwdArgs a) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= a.n) return;
    const int L = a.L;

    // ---- merge this Gaussian's entries in entry (bucket) order (rasterizer.cpp:435-455)
    double acc[kGradVals];
    for (int q = 0; q < kGradVals; ++q) acc[q] = 0.0;
    double rho_grad[64];
    const int Lg = L < 64 ? L : 64;
    for (int l = 0; l < Lg; ++l) rho_grad[l] = 0.0;
    const unsigned cnt = a.count[i];
    if (cnt > 0) {
        const int4 r = a.rect[i];
        const unsigned area = static_cast<unsigned>((r.y - r.x) * (r.w - r.z));
        unsigned long long planes = a.soft ? a.pmask[i] : 0ull;
        int l = a.soft ? -1 : a.plane[i];
        const float* eg = a.egrad + static_cast<size_t>(a.goff[i]) * kGradVals;
        for (unsigned k = 0; k < cnt; ++k, eg += kGradVals) {
            if (a.soft && k % area == 0) {  // next assigned plane
                l = __ffsll(static_cast<long long>(planes)) - 1;
                planes &= planes - 1;
            }
            for (int q = 0; q < kGradVals; ++q) acc[q] += static_cast<double>(eg[q]);
            if (l >= 0 && l < 64) rho_grad[l] += static_cast<double>(eg[kGRho]);
        }
    }

    // ---- straight-through (or relaxed) route to the plane logits (:470-482)
    const double* lg = a.plane_logits + i * L;
    const double tau = a.soft ? a.soft_tau : a.ste_tau;
    int best = 0;
    for (int l = 1; l < L; ++l)
        if (lg[l] > lg[best]) best = l;
    const double top = lg[best];
    double denom = 0.0;
    for (int l = 0; l < L; ++l) denom += exp((lg[l] - top) / tau);
    double dot = 0.0;
    if (a.soft)
        for (int l = 0; l < Lg; ++l) dot += exp((lg[l] - top) / tau) / denom * rho_grad[l];
    if (a.g.plane_logits)
        for (int l = 0; l < L; ++l) {
            const double rg = l < 64 ? rho_grad[l] : 0.0;
            if (!a.soft && rg == 0.0) {  // rg * w = 0 exactly: skip the exponential
                a.g.plane_logits[i * L + l] = 0.0;
                continue;
            }
            const double w = exp((lg[l] - top) / tau) / denom;
            a.g.plane_logits[i * L + l] = a.soft ? w * (rg - dot) / a.soft_tau : rg * w;
        }

    // ---- projection, recomputed in f64 (rasterizer.cpp:10-70)
    const double* W = a.cam.wc;
    const double* xw = a.positions + 3 * i;
    const double d0 = xw[0] - a.cam.pos[0], d1 = xw[1] - a.cam.pos[1], d2 = xw[2] - a.cam.pos[2];
    const double xc = (W[0] * d0 + W[1] * d1) + W[2] * d2;
    const double yc = (W[3] * d0 + W[4] * d1) + W[5] * d2;
    const double zc = (W[6] * d0 + W[7] * d1) + W[8] * d2;
    const double* qv = a.rotations + 4 * i;
    const double* ls = a.log_scales + 3 * i;
    const double qn = sqrt(((qv[0] * qv[0] + qv[1] * qv[1]) + qv[2] * qv[2]) + qv[3] * qv[3]);
    const double qw = qv[0] / qn, qx = qv[1] / qn, qy = qv[2] / qn, qz = qv[3] / qn;
    const double R[9] = {
        1.0 - 2.0 * (qy * qy + qz * qz), 2.0 * (qx * qy - qw * qz),       2.0 * (qx * qz + qw * qy),
        2.0 * (qx * qy + qw * qz),       1.0 - 2.0 * (qx * qx + qz * qz), 2.0 * (qy * qz - qw * qx),
        2.0 * (qx * qz - qw * qy),       2.0 * (qy * qz + qw * qx),       1.0 - 2.0 * (qx * qx + qy * qy),
    };
    const double s3[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
    double Mq[9], Sig[9];
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) Mq[r * 3 + k] = R[r * 3 + k] * s3[k];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            Sig[r * 3 + c] = (Mq[r * 3 + 0] * Mq[c * 3 + 0] + Mq[r * 3 + 1] * Mq[c * 3 + 1]) + Mq[r * 3 + 2] * Mq[c * 3 + 2];
    if (!(zc > a.near_clip)) return;
    const double f = a.cam.focal, iz = 1.0 / zc;
    double J[6] = {f * iz, 0.0, -f * xc * iz * iz, 0.0, f * iz, -f * yc * iz * iz};
    double M[6], Tm[6];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c)
            M[r * 3 + c] = (J[r * 3 + 0] * W[0 * 3 + c] + J[r * 3 + 1] * W[1 * 3 + c]) + J[r * 3 + 2] * W[2 * 3 + c];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c)
            Tm[r * 3 + c] = (M[r * 3 + 0] * Sig[0 * 3 + c] + M[r * 3 + 1] * Sig[1 * 3 + c]) + M[r * 3 + 2] * Sig[2 * 3 + c];
    const double cov00 = ((Tm[0] * M[0] + Tm[1] * M[1]) + Tm[2] * M[2]) + a.dilation;
    const double cov01 = (Tm[0] * M[3] + Tm[1] * M[4]) + Tm[2] * M[5];
    const double cov11 = ((Tm[3] * M[3] + Tm[4] * M[4]) + Tm[5] * M[5]) + a.dilation;
    const double det = cov00 * cov11 - cov01 * cov01;
    if (!(det > 0.0 && isfinite(det))) return;
    const double x = a.opacity_logits[i];
    const double alpha = x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
    if (a.alpha_floor > 0.0 && !(alpha > a.alpha_floor)) return;  // not valid: zero gradients
    const double inv00 = cov11 / det, inv01 = -cov01 / det, inv11 = cov00 / det;

    // ---- chain (rasterizer.cpp:484-525)
    if (a.g.mu_screen) {
        a.g.mu_screen[2 * i] = acc[kGMuX];
        a.g.mu_screen[2 * i + 1] = acc[kGMuY];
    }
    for (int c = 0; c < 3; ++c) {
        if (a.g.amplitudes) a.g.amplitudes[3 * i + c] = acc[kGAmp + c];
        if (a.g.phases) a.g.phases[3 * i + c] = acc[kGPh + c];
    }
    if (a.g.opacity_logits) a.g.opacity_logits[i] = acc[kGAlpha] * alpha * (1.0 - alpha);

    // gcov2 = -inv ginv inv, ginv = [[g00, g01/2], [g01/2, g11]]
    const double gi00 = acc[kGI00], gi01 = 0.5 * acc[kGI01], gi11 = acc[kGI11];
    const double A00 = inv00 * gi00 + inv01 * gi01, A01 = inv00 * gi01 + inv01 * gi11;
    const double A10 = inv01 * gi00 + inv11 * gi01, A11 = inv01 * gi01 + inv11 * gi11;
    const double gc[4] = {-(A00 * inv00 + A01 * inv01), -(A00 * inv01 + A01 * inv11),
                          -(A10 * inv00 + A11 * inv01), -(A10 * inv01 + A11 * inv11)};
    // gsigma = M^T gcov2 M
    double gsig[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0.0;
            for (int p = 0; p < 2; ++p)
                for (int q = 0; q < 2; ++q) s += M[p * 3 + r] * gc[p * 2 + q] * M[q * 3 + c];
            gsig[r * 3 + c] = s;
        }
    // covariance_backward (scene.cpp:84-121)
    {
        double dM[9];  // (G + G^T) Mq
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                double s = 0.0;
                for (int k = 0; k < 3; ++k) s += (gsig[r * 3 + k] + gsig[k * 3 + r]) * Mq[k * 3 + c];
                dM[r * 3 + c] = s;
            }
        if (a.g.log_scales)
            for (int k = 0; k < 3; ++k) {
                const double ds = (dM[0 * 3 + k] * R[0 * 3 + k] + dM[1 * 3 + k] * R[1 * 3 + k]) + dM[2 * 3 + k] * R[2 * 3 + k];
                a.g.log_scales[3 * i + k] = ds * s3[k];
            }
        double dR[9];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) dR[r * 3 + k] = dM[r * 3 + k] * s3[k];
        const double dw[9] = {0, -qz, qy, qz, 0, -qx, -qy, qx, 0};
        const double dxm[9] = {0, qy, qz, qy, -2 * qx, -qw, qz, qw, -2 * qx};
        const double dym[9] = {-2 * qy, qx, qw, qx, 0, qz, -qw, qz, -2 * qy};
        const double dzm[9] = {-2 * qz, -qw, qx, qw, -2 * qz, qy, qx, qy, 0};
        double gu[4] = {0, 0, 0, 0};
        for (int t = 0; t < 9; ++t) {
            gu[0] += dR[t] * dw[t];
            gu[1] += dR[t] * dxm[t];
            gu[2] += dR[t] * dym[t];
            gu[3] += dR[t] * dzm[t];
        }
        for (int t = 0; t < 4; ++t) gu[t] *= 2.0;
        const double qnv[4] = {qw, qx, qy, qz};
        const double proj = ((qnv[0] * gu[0] + qnv[1] * gu[1]) + qnv[2] * gu[2]) + qnv[3] * gu[3];
        if (a.g.rotations)
            for (int t = 0; t < 4; ++t) a.g.rotations[4 * i + t] = (gu[t] - qnv[t] * proj) / qn;
    }
    // centre: through the projected mean and the Jacobian (:507-522)
    if (a.g.positions) {
        double gM[6];  // (gcov2 + gcov2^T) M Sigma
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c) {
                double s = 0.0;
                for (int p = 0; p < 2; ++p) {
                    const double gs = gc[r * 2 + p] + gc[p * 2 + r];
                    double ms = 0.0;
                    for (int k = 0; k < 3; ++k) ms += M[p * 3 + k] * Sig[k * 3 + c];
                    s += gs * ms;
                }
                gM[r * 3 + c] = s;
            }
        double gJ[6];  // gM W^T
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c) gJ[r * 3 + c] = (gM[r * 3 + 0] * W[c * 3 + 0] + gM[r * 3 + 1] * W[c * 3 + 1]) + gM[r * 3 + 2] * W[c * 3 + 2];
        const double mx = acc[kGMuX], my = acc[kGMuY];
        double gxc[3] = {J[0] * mx + J[3] * my, J[1] * mx + J[4] * my, J[2] * mx + J[5] * my};
        const double fiz2 = -f * iz * iz;
        gxc[0] += gJ[2] * fiz2;
        gxc[1] += gJ[5] * fiz2;
        gxc[2] += (gJ[0] + gJ[4]) * fiz2 + gJ[2] * (2.0 * f * xc * iz * iz * iz) + gJ[5] * (2.0 * f * yc * iz * iz * iz);
        for (int d = 0; d < 3; ++d) a.g.positions[3 * i + d] = (W[0 * 3 + d] * gxc[0] + W[1 * 3 + d] * gxc[1]) + W[2 * 3 + d] * gxc[2];
    }
}

template <int TILE, int C>
void launch_bwd_c(holo_ctx* ctx, const RasterBwdArgs& a, dim3 grid) {
    constexpr size_t kPart = sizeof(float) * (TILE * TILE / 32) * (TILE == 32 ? 32 : 128) * kGradVals;
    static bool done[256] = {};  // function attributes are per device
    int dev = 0;
    HC_CUDA(cudaGetDevice(&dev));
    if (!done[dev & 255]) {
        HC_CUDA(cudaFuncSetAttribute(k_raster_bwd<TILE, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kPart)));
        done[dev & 255] = true;
    }
    k_raster_bwd<TILE, C><<<grid, TILE * TILE, kPart, ctx->stream>>>(a);
}

template <int TILE>
void launch_raster_bwd_tile(holo_ctx* ctx, const RasterBwdArgs& a) {
    const int tiles_y = a.num_tiles / a.tiles_x;
    const dim3 grid(a.tiles_x, tiles_y, a.num_buckets / a.num_tiles);
    switch (a.C) {
        case 1: launch_bwd_c<TILE, 1>(ctx, a, grid); break;
        case 2: launch_bwd_c<TILE, 2>(ctx, a, grid); break;
        case 3: launch_bwd_c<TILE, 3>(ctx, a, grid); break;
        default: throw Error(HOLO_ERR_CONFIG, "render supports 1 to 3 wavelength channels");
    }
    HC_LAUNCHED(ctx);
}

}  // namespace

void bwd_seed(holo_ctx* ctx, const cx<float>* rep, const float* gi, const double* gi64, cx<float>* gv, size_t n) {
    if (n == 0) return;
    const size_t blocks = (n + 255) / 256;
    const unsigned nb = static_cast<unsigned>(blocks < 8192 ? blocks : 8192);
    if (gi64)
        k_bwd_seed<double><<<nb, 256, 0, ctx->stream>>>(rep, gi64, gv, n);
    else
        k_bwd_seed<float><<<nb, 256, 0, ctx->stream>>>(rep, gi, gv, n);
    HC_LAUNCHED(ctx);
}

void bwd_prep(holo_ctx* ctx, size_t N, const double* amplitudes, const double* phases, const GRec* rec,
              BwdRec* out) {
    if (N == 0) return;
    k_bwd_prep<<<static_cast<unsigned>((N + 255) / 256), 256, 0, ctx->stream>>>(amplitudes, phases, rec, N, out);
    HC_LAUNCHED(ctx);
}

void raster_backward_entries(holo_ctx* ctx, const RasterBwdArgs& a, int tile) {
    if (a.num_buckets <= 0) return;
    switch (tile) {
        case 8: launch_raster_bwd_tile<8>(ctx, a); break;
        case 16: launch_raster_bwd_tile<16>(ctx, a); break;
        case 32: launch_raster_bwd_tile<32>(ctx, a); break;
        default: throw Error(HOLO_ERR_CONFIG, "render supports tile sizes 8, 16 and 32");
    }
}

void gauss_backward(holo_ctx* ctx, const GaussBwdArgs& a) {
    if (a.n == 0) return;
    k_bwd_gauss<<<static_cast<unsigned>((a.n + 255) / 256), 256, 0, ctx->stream>>>(a);
    HC_LAUNCHED(ctx);
}

}  // namespace holo_cuda
