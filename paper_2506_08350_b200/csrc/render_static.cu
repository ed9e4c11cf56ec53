// Render-path propagation with compile-time FFT plans (sm_100a, fp32).
//
// pipeline_forward's propagation (forward_record + inverse_propagate,
// proj/src/propagation.cpp:103-123) as three passes over HBM:
//   1. k_col_fwd      column FFT of every raster layer, in place
//   2. k_row_fused    per row (c, y): row FFT of each plane, times H_{Z_l}, summed
//                     into the spectrum S held in registers; then for every output
//                     (the hologram and each replayed plane) S . M_o -> row IFFT
//                     with M_o = 1 or conj(H_{Z_l}) = H_{-Z_l}
//   3. k_col_inv_epi  column IFFT of each output with the epilogue: hologram
//                     x 1/(w h); intensity |v / (w h)|^2; optional replayed field
// S never exists as a full field unless the planes are sharded across GPUs
// (modes SPEC / REPLAY of k_row_fused bracket the all-reduce of S).  The
// identity FFT2(hologram) = S (the hologram is IFFT2(S)) removes the forward
// transform of inverse_propagate.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "bulk.cuh"
#include "fft_static.cuh"
#include "kernels.cuh"

namespace holo_cuda {

namespace {

using namespace bulk;

template <int N>
struct PlanOf;
// the column IFFT's plan: the forward plan reversed unless specialised (the row
// pass needs the exact reverse to keep its spectrum in registers; the column
// passes are separate kernels)
template <int N>
struct InvColPlanOf;
template <> struct PlanOf<48> { using type = Radices<16, 3>; };
template <> struct PlanOf<64> { using type = Radices<16, 4>; };
template <> struct PlanOf<128> { using type = Radices<16, 8>; };
template <> struct PlanOf<256> { using type = Radices<16, 16>; };
template <> struct PlanOf<512> { using type = Radices<8, 8, 8>; };
// measured at C4 (row pass / column FFT / column IFFT, ms): [16,16,4] 0.136 / 0.069 / 0.078,
// [16,8,8] 0.112 / 0.069 / 0.076, [8,16,8] 0.125 / 0.068 / 0.078, [8,8,16] 0.142 / 0.077 / 0.076
#ifndef HOLO_P1024_A
#define HOLO_P1024_A 16
#define HOLO_P1024_B 8
#define HOLO_P1024_C 8
#endif
template <> struct PlanOf<1024> { using type = Radices<HOLO_P1024_A, HOLO_P1024_B, HOLO_P1024_C>; };
// HOLO_P1080_{A,B,C} / HOLO_P1920_{A,B,C}: plan orderings for measurement
// measured at C3 (column FFT / IFFT, ms): [8,9,15] 0.197 / 0.208, [9,8,15] 0.185 / 0.203,
// [12,9,10] 0.193 / 0.205, [8,15,9] 0.208 / 0.208, [15,9,8] 0.199 / 0.232
#ifndef HOLO_P1080_A
#define HOLO_P1080_A 9
#define HOLO_P1080_B 8
#define HOLO_P1080_C 15
#endif
template <> struct PlanOf<1080> { using type = Radices<HOLO_P1080_A, HOLO_P1080_B, HOLO_P1080_C>; };
// HOLO_ROW1920 selects the 1920-point plan and row-pass shape (tuning).  Measured
// row pass at C3: 1 = [16,8,15], 2 rows x 256 threads, 2 CTAs/SM: 0.451 ms;
// 2 = [16,15,8] 1 row, 3 CTAs: 0.554; 3 = 2 rows x 512: 0.566; 4 = 4 CTAs: 0.626.
// Splitting the pass in two kernels around S in HBM (forward + sum, then the
// replays at higher occupancy) measured 0.465 ms at 2 + 2 CTAs/SM, 0.484 at
// 2 + 3, 0.515 at 3 + 3 and 0.58-0.61 with 1-row replay CTAs at 4/SM, against
// 0.435 fused: occupancy is not what limits this pass.  One row per CTA of 128
// threads (4 or 3 CTAs/SM, same registers per thread): 0.498 ms.
#ifndef HOLO_ROW1920
#define HOLO_ROW1920 1
#endif
// measured at C3 (row pass, ms): [16,8,15] 0.306, [8,15,16] 0.293, [8,16,15] 0.297,
// [15,8,16] 0.318, [15,16,8] 0.314
#ifndef HOLO_P1920_A
#if HOLO_ROW1920 == 1
#define HOLO_P1920_A 8
#define HOLO_P1920_B 15
#define HOLO_P1920_C 16
#else
#define HOLO_P1920_A 16
#define HOLO_P1920_B 15
#define HOLO_P1920_C 8
#endif
#endif
template <> struct PlanOf<1920> { using type = Radices<HOLO_P1920_A, HOLO_P1920_B, HOLO_P1920_C>; };
#ifndef HOLO_P2048_A
#define HOLO_P2048_A 16
#define HOLO_P2048_B 16
#define HOLO_P2048_C 8
#endif
template <> struct PlanOf<2048> { using type = Radices<HOLO_P2048_A, HOLO_P2048_B, HOLO_P2048_C>; };
#ifndef HOLO_P2160_A
#define HOLO_P2160_A 16
#define HOLO_P2160_B 9
#define HOLO_P2160_C 15
#endif
template <> struct PlanOf<2160> { using type = Radices<HOLO_P2160_A, HOLO_P2160_B, HOLO_P2160_C>; };
// measured at C5 (row pass, ms): [16,16,15] 2.120, [16,15,16] 2.090, [15,16,16] 2.184
#ifndef HOLO_P3840_A
#define HOLO_P3840_A 16
#define HOLO_P3840_B 15
#define HOLO_P3840_C 16
#endif
template <> struct PlanOf<3840> { using type = Radices<HOLO_P3840_A, HOLO_P3840_B, HOLO_P3840_C>; };

template <int N>
struct InvColPlanOf {
    using type = typename RevPlan<typename PlanOf<N>::type>::type;
};
// measured at C3 (column IFFT): [15,8,9] (the reverse of [9,8,15]) 0.203 ms, [10,12,9] 0.192 ms
template <> struct InvColPlanOf<1080> { using type = Radices<10, 12, 9>; };
// measured at C5 (column FFT / IFFT, ms): [16,9,15] 1.698 / 2.141 (its reverse), inverse [16,15,9] 1.883
template <> struct InvColPlanOf<2160> { using type = Radices<16, 15, 9>; };

// column passes: strips of NB columns, NT threads, MINB CTAs per SM (register cap)
// The twiddle table is copied to shared memory behind the FFT work area
// (HOLO_COL_SMEM_TW=0 reads it from global memory instead).
#ifndef HOLO_COL_SMEM_TW
#define HOLO_COL_SMEM_TW 0  // measured: global (L1) twiddles 0.211 -> 0.197 ms (col fwd, C3)
#endif
// the row pass's twiddles: shared-memory copy (1) or global / L1 (0); measured at
// C3 with the [8,15,16] plan: 0.292 ms (shared) vs 0.281 ms (L1)
#ifndef HOLO_ROW_SMEM_TW
#define HOLO_ROW_SMEM_TW 0
#endif
template <int H_, int NB_, int NT_, int MINB_>
struct ColCfgT {
    static constexpr int H = H_, NB = NB_, NT = NT_, kMinBlocks = MINB_;
    using B = Batch<H, NB, NT>;
    static constexpr int kWorkF = FftSmem<B, typename PlanOf<H>::type>::kElems;
    static constexpr int kWorkI = FftSmem<B, typename InvColPlanOf<H>::type>::kElems;
    static constexpr int kWorkElems = kWorkF > kWorkI ? kWorkF : kWorkI;
    static constexpr size_t kSmem = sizeof(cx<float>) * (kWorkElems + (HOLO_COL_SMEM_TW ? H : 0));
};

// twiddles for a column pass: staged into shared memory before the first stage
// (whose closing barrier publishes them; stage 1 uses none)
template <class Cfg>
__device__ __forceinline__ const cx<float>* col_twiddles(cx<float>* sm, const cx<float>* __restrict__ tw) {
    if constexpr (HOLO_COL_SMEM_TW) {
        cx<float>* s_tw = sm + Cfg::kWorkElems;
        for (int k = threadIdx.x; k < Cfg::H; k += Cfg::NT) s_tw[k] = tw[k];
        return s_tw;
    }
    return tw;
}
// default: 8-column strips (64-byte row segments); 2 CTAs per SM while 64 registers suffice
// (HOLO_COL_NB / _NT / _MINB override the shape, for measurement)
#ifndef HOLO_COL_NB
#define HOLO_COL_NB 8
#endif
#ifndef HOLO_COL_NT
#define HOLO_COL_NT 0
#endif
#ifndef HOLO_COL_MINB
#define HOLO_COL_MINB 0
#endif
template <int H>
using ColCfg = ColCfgT<H, HOLO_COL_NB, (HOLO_COL_NT ? HOLO_COL_NT : (H >= 1024 ? 512 : 256)),
                       (HOLO_COL_MINB ? HOLO_COL_MINB : (H <= 1280 ? 2 : 1))>;

// row pass: NBR rows of one channel per CTA
template <int W_, int NBR_, int NT_, int MINB_>
struct RowCfgT {
    static constexpr int W = W_, NBR = NBR_, NT = NT_, kMinBlocks = MINB_;
    using B = Batch<W, NBR, NT>;
};
template <int W>
struct RowCfgSel {
    using type = RowCfgT<W, (W <= 512 ? 4 : (W <= 2048 ? 2 : 1)), (W >= 1024 ? 256 : 128), 2>;
};
#if HOLO_ROW1920 == 2
template <> struct RowCfgSel<1920> { using type = RowCfgT<1920, 1, 256, 3>; };
#elif HOLO_ROW1920 == 3
template <> struct RowCfgSel<1920> { using type = RowCfgT<1920, 2, 512, 1>; };
#elif HOLO_ROW1920 == 4
template <> struct RowCfgSel<1920> { using type = RowCfgT<1920, 1, 256, 4>; };
#endif
template <int W>
using RowCfg = typename RowCfgSel<W>::type;

__device__ __forceinline__ cx<float> czf() { return mk(0.0f, 0.0f); }

// e^{i theta} for |theta| up to a few thousand rad: two-constant reduction into
// [-pi, pi] then the MUFU sin/cos (abs. error <= 2^-21.4 there).
__device__ __forceinline__ cx<float> phasor_reduced(float theta) {
    const float k = rintf(theta * 0.159154943091895336f);
    float red = fmaf(-k, 6.28318548202514648f, theta);  // 2 pi rounded to float
    red = fmaf(-k, -1.74845553e-07f, red);              // minus (2 pi - that)
    float s, c;
    __sincosf(red, &s, &c);
    return mk(c, s);
}

// ---------------------------------------------------------------- 1. column FFT (forward, in place)

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT, Cfg::kMinBlocks) k_col_fwd(cx<float>* __restrict__ data, int W,
                                                                      const cx<float>* __restrict__ tw) {
    constexpr int H = Cfg::H;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<float>* sm = reinterpret_cast<cx<float>*>(smem_raw);
    const int x0 = blockIdx.x * Cfg::NB;
    cx<float>* base = data + static_cast<size_t>(blockIdx.y) * H * W;
    auto load = [&](int, int, int b, int i) -> cx<float> {
        const int x = x0 + b;
        return x < W ? base[static_cast<size_t>(i) * W + x] : czf();
    };
    auto store = [&](int, int, int b, int i, cx<float> v) {
        const int x = x0 + b;
        if (x < W) base[static_cast<size_t>(i) * W + x] = v;
    };
    fft_static<float, -1, typename Cfg::B, typename PlanOf<H>::type>(sm, col_twiddles<Cfg>(sm, tw), load, store);
}

// ---------------------------------------------------------------- 2. row pass with the spectrum in registers

// Row-pass shared memory: FFT work area; the prefetch buffer for the next plane's
// NBR rows (each row padded by 8 complex = 16 banks; FULL / SPEC); the twiddle
// table; per owned spectral sample ([slot][thread], conflict-free) either the
// plane-independent TF factor G (DIRECT) or the plane-to-plane TF ratio Q; the
// per-plane TF constants.
template <class Cfg, int MODE, bool DIRECT>
struct RowSmem {
    using LS = LastStage<typename Cfg::B, typename PlanOf<Cfg::W>::type>;
    static constexpr int kRowPad = Cfg::W + 8;
    static constexpr size_t kWork = sizeof(cx<float>) * FftSmem<typename Cfg::B, typename PlanOf<Cfg::W>::type>::kElems;
    static constexpr size_t kPre = MODE == kModeReplay ? 0 : sizeof(cx<float>) * Cfg::NBR * kRowPad;
    static constexpr size_t kG = (DIRECT ? sizeof(float) : sizeof(cx<float>)) * LS::kBPT * LS::kR * Cfg::NT;
    // the twiddle table is copied to shared memory only while kMinBlocks CTAs still
    // fit an SM (227 KB); wide rows (3840) read it through L1 instead
    static constexpr bool kTwSmem =
        HOLO_ROW_SMEM_TW && (kWork + kPre + sizeof(cx<float>) * Cfg::W + kG + 2048) * Cfg::kMinBlocks <= 227 * 1024;
    static constexpr size_t kTw = kTwSmem ? sizeof(cx<float>) * Cfg::W : 0;
    static constexpr size_t kTf = kWork + kPre + kTw + kG;  // offset of the per-plane constants
    static size_t bytes(int Lloc) { return kTf + sizeof(float2) * (Lloc > 0 ? Lloc : 1); }
};

// The planes are evenly spaced (plane_positions, wave_config.cpp:18-30), so the
// transfer functions of consecutive planes differ by one per-sample factor:
//   H_l = A Q^l,  A = e^{i (phase0_0 - 2 pi z_0 g)},  Q = e^{i (dphase - 2 pi dz g)}
// (g = f^2 / (1/l + sqrt(1/l^2 - f^2)) as in tf_value<float>; dphase = 2 pi dz / lambda
// reduced mod 2 pi in f64 on the host).  The forward sum is evaluated by Horner over
// the planes in reverse order, S' = X_{L-1}, S' = Q S' + X_l, S = A S' -- one complex
// FMA per plane and sample instead of a range-reduced sin / cos -- and the replays
// take S conj(H_l) = S' conj(Q)^l, stepping S' by conj(Q) after each plane.  DIRECT
// evaluates every H_l itself (local band limits, unevenly spaced planes).
template <class Cfg, int MODE, bool DIRECT>
__global__ void __launch_bounds__(Cfg::NT, Cfg::kMinBlocks) k_row_fused(
    const cx<float>* __restrict__ layers,  // [Lloc][C][H][W], column-transformed (FULL, SPEC)
    cx<float>* __restrict__ spec,          // [C][H][W]: written (SPEC) or read (REPLAY)
    cx<float>* __restrict__ out,           // [O][C][H][W] row-inverse-transformed outputs (FULL, REPLAY)
    int H, int C, int Lloc, int has_holo, int nrep, const TfChan* __restrict__ tfc,
    const double* __restrict__ fx, const double* __restrict__ fy, const cx<float>* __restrict__ tw, int row_base,
    const cx<float>* __restrict__ qtab) {
    constexpr int W = Cfg::W;
    constexpr int NBR = Cfg::NBR;
    using B = typename Cfg::B;
    using P = typename PlanOf<W>::type;
    using Pinv = typename RevPlan<P>::type;
    using LS = LastStage<B, P>;
    using SM = RowSmem<Cfg, MODE, DIRECT>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<float>* sm = reinterpret_cast<cx<float>*>(smem_raw);
    cx<float>* pre = reinterpret_cast<cx<float>*>(smem_raw + SM::kWork);
    const cx<float>* s_tw = SM::kTwSmem ? reinterpret_cast<cx<float>*>(smem_raw + SM::kWork + SM::kPre) : tw;
    unsigned char* s_slot = smem_raw + SM::kWork + SM::kPre + SM::kTw;
    float2* s_tf = reinterpret_cast<float2*>(smem_raw + SM::kTf);  // (phase0, 2 pi z) per plane
    __shared__ unsigned long long s_bar;

    // row = c * H + y; a CTA never spans two channels.  row_base = c0 * H restricts a
    // launch to the channels [c0, c0 + gridDim.x * NBR / H) (per-channel pipelines
    // of a plane-sharded frame).
    const int row0 = row_base + blockIdx.x * NBR;
    const int c = row0 / H;
    const size_t plane_stride = static_cast<size_t>(C) * H * W;
    const int nplanes = MODE == kModeReplay ? nrep : Lloc;
    for (int l = threadIdx.x; l < nplanes; l += Cfg::NT) s_tf[l] = make_float2(tfc[l * C + c].phase0, tfc[l * C + c].two_pi_z_f);
    if constexpr (SM::kTwSmem)
        for (int k = threadIdx.x; k < W; k += Cfg::NT) const_cast<cx<float>*>(s_tw)[k] = tw[k];

    // prefetch of plane l's NBR rows (one thread issues; the buffer is free once
    // every thread has finished the previous plane's first FFT stage)
    auto issue = [&](int l) {
        const cx<float>* src = layers + l * plane_stride + static_cast<size_t>(row0) * W;
        fence_proxy_async_smem();  // the buffer's previous generic reads precede the async writes
        mbar_expect_tx(&s_bar, NBR * W * static_cast<unsigned>(sizeof(cx<float>)));
#pragma unroll
        for (int b = 0; b < NBR; ++b)
            bulk_g2s(pre + b * SM::kRowPad, src + static_cast<size_t>(b) * W,
                     W * static_cast<unsigned>(sizeof(cx<float>)), &s_bar);
    };
    // forward planes in the order the sum needs them: Horner runs from the last plane
    auto fwd_plane = [&](int it) { return DIRECT ? it : Lloc - 1 - it; };
    if constexpr (MODE != kModeReplay) {
        if (threadIdx.x == 0) {
            mbar_init(&s_bar, 1);
            mbar_init_fence();
        }
        __syncthreads();
        if (threadIdx.x == 0 && Lloc > 0) issue(fwd_plane(0));
    } else {
        __syncthreads();
    }

    // (q, r) <-> (b, i) of the last forward stage = first inverse stage
    auto owner = [&](int q, int r, int& b, int& i) -> bool {
        constexpr int M = W / LS::kR;
        const int t = threadIdx.x + q * B::kNT;
        b = t % B::kNB;
        i = t / B::kNB + r * M;
        return t < M * B::kNB;
    };
    // g = f^2 / (1/l + sqrt(1/l^2 - f^2)) at owned sample (q, r), or -1 outside the
    // propagating band (band test in f64, reference order)
    const TfChan p0 = tfc[c];  // 1/l^2, 1/l depend on the channel only
    auto g_at = [&](int q, int r) -> float {
        int b, i;
        float g = -1.0f;
        if (owner(q, r, b, i)) {
            const double fxv = fx[i], fyv = fy[(row0 + b) - c * H];
            const double fx2 = __dmul_rn(fxv, fxv), fy2 = __dmul_rn(fyv, fyv);
            const double arg = __dsub_rn(__dsub_rn(p0.inv_l2, fx2), fy2);
            if (!(arg < 0.0)) g = static_cast<float>(__dadd_rn(fx2, fy2)) / (p0.inv_l + sqrtf(static_cast<float>(arg)));
        }
        return g;
    };
    // A = H_{plane 0} (for the Horner form)
    // A = 1 exactly when the first plane sits at z = 0 (every unsharded frame at the
    // paper's optics: Z_0 = 0 for L >= 2, wave_config.cpp:18-30) -- then S = S'
    const bool a_one = s_tf[0].x == 0.0f && s_tf[0].y == 0.0f;
    auto a_at = [&](int q, int r) -> cx<float> {
        const float2 t = s_tf[0];
        return phasor_reduced(t.x - t.y * g_at(q, r));
    };

    cx<float> S[LS::kBPT][LS::kR];
    // DIRECT: G per slot; otherwise Q per slot (0 outside the band)
    auto G = [&](int q, int r) -> float& {
        return reinterpret_cast<float*>(s_slot)[(q * LS::kR + r) * Cfg::NT + threadIdx.x];
    };
    auto Qs = [&](int q, int r) -> cx<float>& {
        return reinterpret_cast<cx<float>*>(s_slot)[(q * LS::kR + r) * Cfg::NT + threadIdx.x];
    };
    {
        // Q of the owned samples from the frame-invariant table (plane_ratio_table)
#pragma unroll
        for (int q = 0; q < LS::kBPT; ++q)
#pragma unroll
            for (int r = 0; r < LS::kR; ++r) {
                S[q][r] = czf();
                if constexpr (DIRECT) {
                    G(q, r) = g_at(q, r);
                } else {
                    int b, i;
                    if (owner(q, r, b, i)) Qs(q, r) = qtab[static_cast<size_t>(row0 + b) * W + i];
                }
            }
    }
    // DIRECT: H_{Z_l} at owned sample (q, r) inside the propagating band: the
    // plane-independent part G and the plane's (phase0, 2 pi z); local band limits
    // (rare) take the full f64 path.  The band mask (H = 0 outside, for every plane)
    // is applied once to S instead of per plane: S = sum_l H_l X_l vanishes there,
    // and so does every S . conj(H_l).
    auto tf = [&](int l, int q, int r, int b, int i) -> cx<float> {
        const TfChan p = tfc[l * C + c];
        if (p.local) return tf_value<float>(p, fx[i], fy[(row0 + b) - c * H]);
        const float2 t = s_tf[l];
        return phasor_reduced(t.x - t.y * G(q, r));
    };
    auto band_mask = [&]() {
#pragma unroll
        for (int q = 0; q < LS::kBPT; ++q)
#pragma unroll
            for (int r = 0; r < LS::kR; ++r) {
                if constexpr (DIRECT) {
                    if (G(q, r) < 0.0f) S[q][r] = czf();
                } else {
                    const cx<float> Q = Qs(q, r);
                    if (Q.x == 0.0f && Q.y == 0.0f) S[q][r] = czf();
                }
            }
    };

    if constexpr (MODE != kModeReplay) {
        for (int it = 0; it < Lloc; ++it) {
            const int l = fwd_plane(it);
            mbar_wait(&s_bar, it & 1);
            auto load = [&](int, int, int b, int i) -> cx<float> { return pre[b * SM::kRowPad + i]; };
            auto store = [&](int q, int r, int b, int i, cx<float> v) {
                if constexpr (DIRECT)
                    S[q][r] = cfma(v, tf(l, q, r, b, i), S[q][r]);
                else
                    S[q][r] = cfma(S[q][r], Qs(q, r), v);  // S' = Q S' + X_l
            };
            // once the first stage has read the buffer, start loading the next plane
            auto hook = [&] {
                if (threadIdx.x == 0 && it + 1 < Lloc) issue(fwd_plane(it + 1));
            };
            fft_static<float, -1, B, P>(sm, s_tw, load, store, hook);
        }
        band_mask();
    }
    if constexpr (MODE == kModeSpec) {
        cx<float>* dst = spec + static_cast<size_t>(row0) * W;
#pragma unroll
        for (int q = 0; q < LS::kBPT; ++q)
#pragma unroll
            for (int r = 0; r < LS::kR; ++r) {
                int b, i;
                if (owner(q, r, b, i))
                    dst[static_cast<size_t>(b) * W + i] = DIRECT || a_one ? S[q][r] : S[q][r] * a_at(q, r);
            }
        return;
    }
    if constexpr (MODE == kModeReplay) {
        // S' = S conj(A) (the replayed planes start at plane 0 of the range)
        const cx<float>* srcs = spec + static_cast<size_t>(row0) * W;
#pragma unroll
        for (int q = 0; q < LS::kBPT; ++q)
#pragma unroll
            for (int r = 0; r < LS::kR; ++r) {
                int b, i;
                if (owner(q, r, b, i)) {
                    const cx<float> v = srcs[static_cast<size_t>(b) * W + i];
                    S[q][r] = DIRECT || nrep == 0 || a_one ? v : v * conj(a_at(q, r));
                }
            }
        band_mask();
    }
    // outputs: [hologram] then planes 0..nrep-1 (output_planes in capi.cu)
    if (has_holo) {
        cx<float>* dst = out + static_cast<size_t>(row0) * W;
        const bool plain = DIRECT || a_one || (MODE == kModeReplay && nrep == 0);  // S itself
        auto load = [&](int q, int r, int, int) -> cx<float> { return plain ? S[q][r] : S[q][r] * a_at(q, r); };
        auto store = [&](int, int, int b, int i, cx<float> v) { dst[static_cast<size_t>(b) * W + i] = v; };
        fft_static<float, +1, B, Pinv>(sm, s_tw, load, store);
    }
    for (int l = 0; l < nrep; ++l) {
        cx<float>* dst = out + (static_cast<size_t>(l + has_holo) * C * H + row0) * W;
        auto load = [&](int q, int r, int b, int i) -> cx<float> {
            if constexpr (DIRECT) {
                return S[q][r] * conj(tf(l, q, r, b, i));
            } else {
                const cx<float> v = S[q][r];  // S' conj(Q)^l
                S[q][r] = v * conj(Qs(q, r));
                return v;
            }
        };
        auto store = [&](int, int, int b, int i, cx<float> v) { dst[static_cast<size_t>(b) * W + i] = v; };
        fft_static<float, +1, B, Pinv>(sm, s_tw, load, store);
    }
}

// The plane-to-plane transfer-function ratio Q = e^{i (dphase - 2 pi dz g)} of every
// spectral sample [C][H][W] (0 outside the propagating band): frame-invariant for a
// grid, optics and plane spacing, so it is built once and cached per context; the
// same operations as the row pass's g_at and phasor_reduced.
__global__ void k_plane_ratio(cx<float>* __restrict__ q, int W, int H, int C, const TfChan* __restrict__ tfc,
                              const double* __restrict__ fx, const double* __restrict__ fy) {
    const size_t n = static_cast<size_t>(C) * H * W;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(k % W), y = static_cast<int>((k / W) % H), c = static_cast<int>(k / (static_cast<size_t>(W) * H));
        const TfChan p0 = tfc[c];
        const double fxv = fx[x], fyv = fy[y];
        const double fx2 = __dmul_rn(fxv, fxv), fy2 = __dmul_rn(fyv, fyv);
        const double arg = __dsub_rn(__dsub_rn(p0.inv_l2, fx2), fy2);
        cx<float> v = czf();
        if (!(arg < 0.0)) {
            const float g = static_cast<float>(__dadd_rn(fx2, fy2)) / (p0.inv_l + sqrtf(static_cast<float>(arg)));
            v = phasor_reduced(p0.step_phase - p0.step_2piz * g);
        }
        q[k] = v;
    }
}

// ---------------------------------------------------------------- 3. column IFFT + epilogue

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT, Cfg::kMinBlocks) k_col_inv_epi(const cx<float>* __restrict__ in, int W,
                                                                          int C, int has_holo, float s,
                                                                          const cx<float>* __restrict__ tw,
                                                                          cx<float>* __restrict__ holo,
                                                                          cx<float>* __restrict__ replayed,
                                                                          float* __restrict__ intens, int c_base) {
    constexpr int H = Cfg::H;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<float>* sm = reinterpret_cast<cx<float>*>(smem_raw);
    const int x0 = blockIdx.x * Cfg::NB;
    const int c = c_base + blockIdx.y, o = blockIdx.z;
    const size_t P = static_cast<size_t>(H) * W;
    const cx<float>* src = in + (static_cast<size_t>(o) * C + c) * P;
    const bool is_holo = has_holo && o == 0;
    const size_t obase = is_holo ? static_cast<size_t>(c) * P : (static_cast<size_t>(o - has_holo) * C + c) * P;
    auto load = [&](int, int, int b, int i) -> cx<float> {
        const int x = x0 + b;
        return x < W ? src[static_cast<size_t>(i) * W + x] : czf();
    };
    auto store = [&](int, int, int b, int i, cx<float> v) {
        const int x = x0 + b;
        if (x >= W) return;
        const size_t at = obase + static_cast<size_t>(i) * W + x;
        v = scale(v, s);
        if (is_holo) {
            holo[at] = v;
        } else {
            if (replayed) replayed[at] = v;
            if (intens) intens[at] = v.x * v.x + v.y * v.y;
        }
    };
    using Pinv = typename InvColPlanOf<H>::type;
    fft_static<float, +1, typename Cfg::B, Pinv>(sm, col_twiddles<Cfg>(sm, tw), load, store);
}

template <class K>
void smem_attr(K kernel, size_t bytes) {
    if (bytes > 48 * 1024)
        HC_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

template <class Cfg>
void launch_col_fwd_cfg(holo_ctx* ctx, cx<float>* data, int W, int nfields) {
    smem_attr(k_col_fwd<Cfg>, Cfg::kSmem);
    const dim3 grid((W + Cfg::NB - 1) / Cfg::NB, nfields);
    k_col_fwd<Cfg><<<grid, Cfg::NT, Cfg::kSmem, ctx->stream>>>(data, W, ctx->twiddle<float>(Cfg::H));
    HC_LAUNCHED(ctx);
}

template <class Cfg>
void launch_col_inv_cfg(holo_ctx* ctx, const cx<float>* in, int W, int C, int nout, int has_holo, cx<float>* holo,
                        cx<float>* rep, float* intens, int c0, int nc) {
    smem_attr(k_col_inv_epi<Cfg>, Cfg::kSmem);
    const dim3 grid((W + Cfg::NB - 1) / Cfg::NB, nc, nout);
    const float s = static_cast<float>(1.0 / (static_cast<double>(W) * Cfg::H));
    k_col_inv_epi<Cfg><<<grid, Cfg::NT, Cfg::kSmem, ctx->stream>>>(in, W, C, has_holo, s,
                                                                   ctx->twiddle<float>(Cfg::H), holo, rep, intens, c0);
    HC_LAUNCHED(ctx);
}

template <class Cfg, int MODE, bool LOCAL>
void launch_row_mode(holo_ctx* ctx, const cx<float>* layers, cx<float>* spec, cx<float>* out, int H, int C, int Lloc,
                     int has_holo, int nrep, const TfChan* tfc, const double* fx, const double* fy, int c0, int nc,
                     const cx<float>* qtab) {
    const dim3 grid(nc * H / Cfg::NBR);
    const int nplanes = MODE == kModeReplay ? nrep : Lloc;
    const size_t smem = RowSmem<Cfg, MODE, LOCAL>::bytes(nplanes);
    HC_CUDA(cudaFuncSetAttribute(k_row_fused<Cfg, MODE, LOCAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    k_row_fused<Cfg, MODE, LOCAL><<<grid, Cfg::NT, smem, ctx->stream>>>(
        layers, spec, out, H, C, Lloc, has_holo, nrep, tfc, fx, fy, ctx->twiddle<float>(Cfg::W), c0 * H, qtab);
    HC_LAUNCHED(ctx);
}

template <class Cfg>
void launch_row_cfg(holo_ctx* ctx, int mode, const cx<float>* layers, cx<float>* spec, cx<float>* out, int H, int C,
                    int Lloc, int has_holo, int nrep, const TfChan* tfc, const double* fx, const double* fy,
                    bool local, int c0, int nc, const cx<float>* qtab) {
#define HC_ROW_MODE(M)                                                                                        \
    (local ? launch_row_mode<Cfg, M, true>(ctx, layers, spec, out, H, C, Lloc, has_holo, nrep, tfc, fx, fy, c0, \
                                           nc, qtab)                                                          \
           : launch_row_mode<Cfg, M, false>(ctx, layers, spec, out, H, C, Lloc, has_holo, nrep, tfc, fx, fy, c0, \
                                            nc, qtab))
    switch (mode) {
        case kModeFull: HC_ROW_MODE(kModeFull); break;
        case kModeSpec: HC_ROW_MODE(kModeSpec); break;
        default: HC_ROW_MODE(kModeReplay); break;
    }
#undef HC_ROW_MODE
}

template <int H>
void launch_col_fwd(holo_ctx* ctx, cx<float>* data, int W, int nfields) {
    launch_col_fwd_cfg<ColCfg<H>>(ctx, data, W, nfields);
}

template <int H>
void launch_col_inv(holo_ctx* ctx, const cx<float>* in, int W, int C, int nout, int has_holo, cx<float>* holo,
                    cx<float>* rep, float* intens, int c0, int nc) {
    launch_col_inv_cfg<ColCfg<H>>(ctx, in, W, C, nout, has_holo, holo, rep, intens, c0, nc);
}

template <int W>
void launch_row(holo_ctx* ctx, int mode, const cx<float>* layers, cx<float>* spec, cx<float>* out, int H, int C,
                int Lloc, int has_holo, int nrep, const TfChan* tfc, const double* fx, const double* fy, bool local,
                int c0, int nc, const cx<float>* qtab) {
    launch_row_cfg<RowCfg<W>>(ctx, mode, layers, spec, out, H, C, Lloc, has_holo, nrep, tfc, fx, fy, local, c0, nc,
                              qtab);
}

// the cached Q table of (grid, channels' wavelengths, pitch, plane step) for tfc's plane 0
const cx<float>* plane_ratio_table(holo_ctx* ctx, int W, int H, int C, const TfChan* tfc, double pitch) {
    // the host copy of the constants upload_tf recorded for tfc (no device read-back)
    const auto rec = ctx->tf_host.find(tfc);
    if (rec == ctx->tf_host.end() || rec->second.size() < static_cast<size_t>(C))
        throw Error(HOLO_ERR_NUMERIC, "row pass: transfer-function constants not on record");
    const TfChan* host = rec->second.data();
    std::string key = "qtab";
    char buf[64];
    std::snprintf(buf, sizeof buf, "|%d|%d|%d|%a", W, H, C, pitch);
    key += buf;
    for (int c = 0; c < C; ++c) {
        std::snprintf(buf, sizeof buf, "|%a|%a|%a", host[c].inv_l2, static_cast<double>(host[c].step_phase),
                      static_cast<double>(host[c].step_2piz));
        key += buf;
    }
    auto it = ctx->tables.find(key);
    if (it != ctx->tables.end()) return static_cast<const cx<float>*>(it->second);
    void* p = nullptr;
    const size_t n = static_cast<size_t>(C) * H * W;
    HC_CUDA(cudaMalloc(&p, sizeof(cx<float>) * n));
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 16 * 148));
    k_plane_ratio<<<blocks, 256, 0, ctx->stream>>>(static_cast<cx<float>*>(p), W, H, C, tfc, ctx->freq(W, pitch),
                                                 ctx->freq(H, pitch));
    HC_LAUNCHED(ctx);
    ctx->tables[key] = p;
    return static_cast<const cx<float>*>(p);
}

#define HC_SIZES(X) X(48) X(64) X(128) X(256) X(512) X(1024) X(1080) X(1920) X(2048) X(2160) X(3840)

bool size_listed(int n) {
#define HC_CASE(N) case N:
    switch (n) {
        HC_SIZES(HC_CASE)
        return true;
        default:
            return false;
    }
#undef HC_CASE
}

int row_nbr(int W) {
#define HC_CASE(N) \
    case N:        \
        return RowCfg<N>::NBR;
    switch (W) {
        HC_SIZES(HC_CASE)
        default:
            return 1;
    }
#undef HC_CASE
}

}  // namespace

bool static_render_supported(int W, int H) {
    return size_listed(W) && size_listed(H) && H % row_nbr(W) == 0;
}

void static_col_fwd(holo_ctx* ctx, cx<float>* data, int W, int H, int nfields) {
    if (nfields <= 0) return;
#define HC_CASE(N)                                    \
    case N:                                           \
        launch_col_fwd<N>(ctx, data, W, nfields);     \
        return;
    switch (H) {
        HC_SIZES(HC_CASE)
        default:
            throw Error(HOLO_ERR_CONFIG, "no static column plan");
    }
#undef HC_CASE
}

void static_col_inv(holo_ctx* ctx, const cx<float>* in, int W, int H, int C, int nout, int has_holo,
                    cx<float>* holo, cx<float>* rep, float* intens, int c0, int nc) {
    if (nc < 0) nc = C - c0;
    if (nout <= 0 || nc <= 0) return;
#define HC_CASE(N)                                                                  \
    case N:                                                                         \
        launch_col_inv<N>(ctx, in, W, C, nout, has_holo, holo, rep, intens, c0, nc); \
        return;
    switch (H) {
        HC_SIZES(HC_CASE)
        default:
            throw Error(HOLO_ERR_CONFIG, "no static column plan");
    }
#undef HC_CASE
}

void static_row(holo_ctx* ctx, int mode, const cx<float>* layers, cx<float>* spec, cx<float>* out, int W, int H,
                int C, int Lloc, int has_holo, int nrep, const TfChan* tfc, double pitch, bool local, int c0, int nc) {
    if (nc < 0) nc = C - c0;
    if (nc <= 0) return;
    const double* fx = ctx->freq(W, pitch);
    const double* fy = ctx->freq(H, pitch);
    const cx<float>* qtab = local ? nullptr : plane_ratio_table(ctx, W, H, C, tfc, pitch);
#define HC_CASE(N)                                                                                              \
    case N:                                                                                                     \
        launch_row<N>(ctx, mode, layers, spec, out, H, C, Lloc, has_holo, nrep, tfc, fx, fy, local, c0, nc, qtab); \
        return;
    switch (W) {
        HC_SIZES(HC_CASE)
        default:
            throw Error(HOLO_ERR_CONFIG, "no static row plan");
    }
#undef HC_CASE
}

}  // namespace holo_cuda
