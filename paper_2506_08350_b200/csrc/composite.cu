// K7 composite: per-(plane, tile) front-to-back complex alpha compositing (sm_100a).
//
// Restates the hot loop of raster_forward (proj/src/rasterizer.cpp:227-261) with
// evaluate() (:124-135): per pixel centre (px + 0.5, py + 0.5), in bucket order,
//   stop once T < term_eps (checked before each entry),
//   a = min(alpha * exp(-form / 2) * rho, alpha_clamp), skip unless a > alpha_floor,
//   acc_c += a T amp_c e^{i phi_c},  T *= 1 - a,  ++n_contrib.
// Bucket order -- ascending (zc, gidx), rasterizer.cpp:221-224 -- is restored
// before compositing: buckets of up to kWarpSortCap entries by k_sort_small / k_sort_large_dev (one
// warp per bucket, shuffle bitonic), buckets above kSortCap by binning.cu, and the
// ones in between by the compositing CTA itself in shared memory.
// Compositing: one CTA per bucket, one thread per pixel.  Records are staged 256
// at a time in shared memory; each warp covers an 8x4 pixel block and, 32
// entries per ballot, skips entries whose accept ellipse (a > alpha_floor) misses
// the block's bounding box, then walks the hits two at a time (the two
// evaluations are independent; only the blend is serial).  Evaluation is fp32
// with the centre offset formed in f64 per entry, so dx, dy keep full fp32
// precision, and alpha folded into the exponent: a = 2^(q + log2 alpha).
#include "raster_eval.cuh"
#include "sort_warp.cuh"

namespace holo_cuda {

namespace {

using namespace warpsort;

template <int TILE>
struct TileGeom {
    static constexpr int kThreads = TILE * TILE;
    // warp block: 8 wide x 4 tall (TILE >= 8); TILE/8 blocks per row
    static constexpr int kBlocksX = TILE / 8;
};

// One warp per bucket of 2..128 entries (129..kWarpSortCap: binning.cu, with the large ones).
// The warp of a larger bucket instead appends it to the device list of the
// mid-size (129..kWarpSortCap: nlist[1], mid) or large (> kSortCap: nlist[0],
// large) buckets that k_sort_large_dev sorts next.  Bucket bounds are clamped to
// the reserved capacity, so at most capacity / 129 resp. capacity / (kSortCap + 1)
// buckets qualify; the list indices are bounded all the same.
#ifndef HOLO_SORT_SMALL_WARPS
#define HOLO_SORT_SMALL_WARPS 8  // warps (buckets) per CTA
#endif
#ifndef HOLO_SORT_SMALL_MINB
#define HOLO_SORT_SMALL_MINB 6  // 40 registers: C3 binning -4 us, C5 -37 us (8: C5 -49, C3/C4 slower)
#endif
__global__ void __launch_bounds__(32 * HOLO_SORT_SMALL_WARPS, HOLO_SORT_SMALL_MINB * 8 / HOLO_SORT_SMALL_WARPS) k_sort_small(const unsigned* __restrict__ bstart, long long B,
                                                    unsigned capacity, const unsigned long long* __restrict__ zkey,
                                                    int* __restrict__ egidx, int* __restrict__ large,
                                                    unsigned max_large, int* __restrict__ mid, unsigned max_mid,
                                                    unsigned* __restrict__ nlist) {
    const long long b = static_cast<long long>(blockIdx.x) * HOLO_SORT_SMALL_WARPS + (threadIdx.x >> 5);
    if (b >= B) return;
    const int lane = threadIdx.x & 31;
    const unsigned e0 = min(bstart[b], capacity);
    const int n = static_cast<int>(min(bstart[b + 1], capacity) - e0);
    if (n > 128) {
        if (lane == 0) {
            if (n > kSortCap) {
                const unsigned k = atomicAdd(nlist, 1u);
                if (k < max_large) large[k] = static_cast<int>(b);
            } else if (n <= kWarpSortCap) {
                const unsigned k = atomicAdd(nlist + 1, 1u);
                if (k < max_mid) mid[k] = static_cast<int>(b);
            }
        }
        return;
    }
    if (n < 2) return;  // warp-uniform
    // 32-bit keys, else 64-bit keys, else the exact (zc, gidx) pairs
    if (n <= 32) {
        if (!warp_sort_bucket_u32<1>(zkey, egidx, e0, n, lane) && !warp_sort_bucket_fast<1>(zkey, egidx, e0, n, lane))
            warp_sort_bucket<1>(zkey, egidx, e0, n, lane);
    } else if (n <= 64) {
        if (!warp_sort_bucket_u32<2>(zkey, egidx, e0, n, lane) && !warp_sort_bucket_fast<2>(zkey, egidx, e0, n, lane))
            warp_sort_bucket<2>(zkey, egidx, e0, n, lane);
    } else if (n <= 128) {
        if (!warp_sort_bucket_u32<4>(zkey, egidx, e0, n, lane) && !warp_sort_bucket_fast<4>(zkey, egidx, e0, n, lane))
            warp_sort_bucket<4>(zkey, egidx, e0, n, lane);
    }
}

#ifdef HOLO_COUNT
__device__ unsigned long long g_counts[4];
#endif

// Buckets of kWarpSortCap + 1 .. kSortCap entries: sorted by the compositing CTA in
// shared memory on (zc, gidx) (rank sort up to 256 entries, bitonic above) into
// s_ord; the sorted gidx are written back so the lists stay in reference order
// for the frame's other consumers (HOLO_BUF_ENTRY_*, the backward pass).
template <int NT>
__device__ __forceinline__ void sort_bucket_cta(const CompositeArgs& a, unsigned e0, int n, int tid,
                                                unsigned long long* key, int* gid, int* s_ord) {
    for (int t = tid; t < n; t += NT) {
        const int g = a.egidx[e0 + t];
        key[t] = a.zkey[g];
        gid[t] = g;
    }
    __syncthreads();
    if (n <= 256) {
        for (int t = tid; t < n; t += NT) {
            const unsigned long long k = key[t];
            const int g = gid[t];
            int rank = 0;
            for (int j = 0; j < n; ++j) {
                const unsigned long long kj = key[j];
                rank += (kj < k || (kj == k && gid[j] < g)) ? 1 : 0;
            }
            s_ord[rank] = g;
        }
    } else {
        int P = 1;
        while (P < n) P <<= 1;
        for (int t = n + tid; t < P; t += NT) {
            key[t] = ~0ull;
            gid[t] = 0x7fffffff;
        }
        __syncthreads();
        for (int k = 2; k <= P; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int t = tid; t < P; t += NT) {
                    const int u = t ^ j;
                    if (u > t) {
                        const bool up = (t & k) == 0;
                        const unsigned long long ka = key[t], kb = key[u];
                        const int ga = gid[t], gb = gid[u];
                        const bool b_less = kb < ka || (kb == ka && gb < ga);
                        const bool a_less = ka < kb || (ka == kb && ga < gb);
                        if (up ? b_less : a_less) {
                            key[t] = kb;
                            key[u] = ka;
                            gid[t] = gb;
                            gid[u] = ga;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int t = tid; t < n; t += NT) s_ord[t] = gid[t];
    }
    __syncthreads();
    for (int t = tid; t < n; t += NT) a.egidx[e0 + t] = s_ord[t];
}

// 16x16 tiles: 7 CTAs (56 warps) per SM, 36 registers -- measured faster than 6 (40 registers,
// -1.3 %), 5 (48 registers) and 8 (32 registers, spills)
#ifndef HOLO_COMP_TEST
#define HOLO_COMP_TEST 2
#endif
#ifndef HOLO_COMP_MINB
#define HOLO_COMP_MINB 7
#endif
// k_composite2 (two pixels per thread) for 16x16 tiles; HOLO_COMP2=0 selects k_composite
#ifndef HOLO_COMP2
#define HOLO_COMP2 1
#endif
#ifndef HOLO_COMP2_MINB
#define HOLO_COMP2_MINB 8
#endif
// unroll factor of k_composite2's walk over a chunk's hits (measurement knob)
#ifndef HOLO_COMP2_UNROLL
#define HOLO_COMP2_UNROLL 4
#endif
// k_composite2's accept predicate as one setp.and + selp per pixel (measurement knob)
#ifndef HOLO_COMP_PRED
#define HOLO_COMP_PRED 1
#endif
// pixels per thread of k_composite2 (2: 128 threads per tile, 4: 64)
#ifndef HOLO_COMP_PPT
#define HOLO_COMP_PPT 2
#endif
#ifndef HOLO_COMP4_MINB
#define HOLO_COMP4_MINB 12
#endif

// AUX: count contributions for n_contrib (HOLO_OUT_AUX); compiled out otherwise
template <int TILE, int C, bool AUX>
__global__ void __launch_bounds__(TILE * TILE, TILE == 16 ? HOLO_COMP_MINB : 1) k_composite(CompositeArgs a) {
    using G = TileGeom<TILE>;
    constexpr int kStage = 256;  // records staged per batch
    constexpr int kTest = HOLO_COMP_TEST;  // box tests per lane per ballot round
    // the mid-size sort's arrays share storage with the staging arrays (the sort
    // finishes, behind a barrier, before the first staging write)
    union Smem {
        struct {
            unsigned long long key[kSortCap];
            int gid[kSortCap];
        } sort;
        struct {
            Staged rec[kStage + 1];  // [kStage]: a record that never accepts (pads odd hit counts)
            float4 box[kStage];      // xlo, xhi, ylo, yhi of the accept ellipse, tile-relative
        } st;
    };
    __shared__ Smem sm;
    __shared__ int s_ord[kSortCap];
    __shared__ __align__(8) int s_hit[G::kThreads / 32][32 * kTest + 2];  // per warp: byte offsets of the chunk's hit records

    const int tx = blockIdx.x, ty = blockIdx.y, lplane = blockIdx.z;  // grid = (tiles_x, tiles_y, planes)
    const int lb = (lplane * gridDim.y + ty) * gridDim.x + tx;        // local bucket
    const int px0 = tx * TILE, py0 = ty * TILE;
    const unsigned e0 = min(a.bstart[lb], a.capacity);
    const int n = static_cast<int>(min(a.bstart[lb + 1], a.capacity) - e0);
    const int plane = a.plane_begin + lplane;

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int bx = (warp % G::kBlocksX) * 8, by = (warp / G::kBlocksX) * 4;
    const int lx = bx + (lane & 7), ly = by + (lane >> 3);
    const int px = px0 + lx, py = py0 + ly;
    const bool inside = px < a.W && py < a.H;
    const float eps = a.term_eps;

    float T = 1.0f;
    int contrib = 0, elast = -1;
    cx<float> acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = mk(0.0f, 0.0f);
    // the reference checks T < term_eps before every entry; T never increases, so
    // "stopped" is exactly !(T >= eps) (outside pixels are parked as stopped)
    bool done = !inside || !(1.0f >= eps);

    if (n > 0) {
        const bool presorted = n <= kWarpSortCap || n > kSortCap;
        if (!presorted) sort_bucket_cta<G::kThreads>(a, e0, n, tid, sm.sort.key, sm.sort.gid, s_ord);

        const float fx = static_cast<float>(lx) + 0.5f, fy = static_cast<float>(ly) + 0.5f;
        const float bxlo = static_cast<float>(bx) + 0.5f, bxhi = static_cast<float>(bx) + 7.5f;
        const float bylo = static_cast<float>(by) + 0.5f, byhi = static_cast<float>(by) + 3.5f;
        // accept = a > alpha_floor, or a > 0 without a positive floor (rasterizer.cpp:133)
        const float thr = a.floor_positive ? a.alpha_floor : 0.0f;
        const float clamp = a.alpha_clamp;

        for (int base = 0; base < n; base += kStage) {
            const int cnt = (n - base) < kStage ? (n - base) : kStage;
            // stage sorted records: tile-relative centre (formed in f64), conic,
            // log2(alpha) (times rho in soft mode), channel phasors, accept box
            for (int t = tid; t < cnt; t += G::kThreads) {
                const int g = presorted ? a.egidx[e0 + base + t] : s_ord[base + t];
                const GRec r = a.rec[g];
                float alpha = r.alpha;
                if (a.soft)
                    alpha = static_cast<float>(static_cast<double>(r.alpha) * a.rho[static_cast<size_t>(g) * a.L + plane]);
                stage_entry(r, px0, py0, alpha, sm.st.rec[t], sm.st.box[t]);
            }
            if (tid == 0) {  // a = 2^-inf = 0: never accepted, and its blend adds exact zeros
                Staged& z = sm.st.rec[kStage];
                z.a = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                z.b = make_float4(0.0f, -INFINITY, 0.0f, 0.0f);
                z.c = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            }
            __syncthreads();
            if (!__all_sync(0xffffffffu, done)) {
                // 32 kTest entries at a time: each lane tests kTest accept boxes against
                // this warp's 8x4 block of pixel centres; the hits are compacted (byte
                // offsets, padded to an even count with the never-accepting record) and
                // the warp walks them in order, two per step, branch-free per lane
                // (predicated accept).
                const char* recs = reinterpret_cast<const char*>(sm.st.rec);
                int* hits = s_hit[warp];
                for (int c0 = 0; c0 < cnt; c0 += 32 * kTest) {
                    const unsigned below = (1u << lane) - 1u;
                    int nh = 0;
#pragma unroll
                    for (int q = 0; q < kTest; ++q) {
                        const int j = c0 + 32 * q + lane;
                        const bool h = j < cnt && box_hits(sm.st.box[j], bxlo, bxhi, bylo, byhi);
                        const unsigned m = __ballot_sync(0xffffffffu, h);
                        if (h) hits[nh + __popc(m & below)] = j * static_cast<int>(sizeof(Staged));
                        nh += __popc(m);
                    }
                    if (lane == 0) hits[nh] = kStage * static_cast<int>(sizeof(Staged));
                    __syncwarp();
#ifdef HOLO_COUNT
                    unsigned long long n_eval = 0, n_any = 0, n_acc = 0;
#endif
                    for (int k = 0; k < nh; k += 2) {
                        const int2 off = *reinterpret_cast<const int2*>(hits + k);
                        const Staged* e0p = reinterpret_cast<const Staged*>(recs + off.x);
                        const Staged* e1p = reinterpret_cast<const Staged*>(recs + off.y);
                        float4 B0, B1;
                        const float al0 = eval_alpha(e0p, fx, fy, clamp, B0);
                        const float al1 = eval_alpha(e1p, fx, fy, clamp, B1);
                        const bool acc0 = (al0 > thr) && (T >= eps);
                        const float w0 = acc0 ? al0 * T : 0.0f;
                        blend<C>(e0p, B0, w0, acc);
                        T -= w0;  // T (1 - a)
                        if constexpr (AUX) {
                            contrib += acc0 ? 1 : 0;
                            elast = acc0 ? base + off.x / static_cast<int>(sizeof(Staged)) : elast;
                        }
                        const bool acc1 = (al1 > thr) && (T >= eps);
                        const float w1 = acc1 ? al1 * T : 0.0f;
                        blend<C>(e1p, B1, w1, acc);
                        T -= w1;
                        if constexpr (AUX) {
                            contrib += acc1 ? 1 : 0;
                            elast = acc1 ? base + off.y / static_cast<int>(sizeof(Staged)) : elast;
                        }
#ifdef HOLO_COUNT
                        n_eval += (k + 1 < nh) ? 2 : 1;
                        n_any += (__ballot_sync(0xffffffffu, acc0) ? 1 : 0) + (__ballot_sync(0xffffffffu, acc1) ? 1 : 0);
                        n_acc += __popc(__ballot_sync(0xffffffffu, acc0)) + __popc(__ballot_sync(0xffffffffu, acc1));
#endif
                    }
                    __syncwarp();  // the next chunk rewrites hits[]
#ifdef HOLO_COUNT
                    if (lane == 0) {
                        atomicAdd(&g_counts[0], n_eval);
                        atomicAdd(&g_counts[1], n_any);
                        atomicAdd(&g_counts[2], n_acc);
                        atomicAdd(&g_counts[3], 1ull);
                    }
#endif
                    done = !inside || !(T >= eps);
                    if (__all_sync(0xffffffffu, done)) break;
                }
            }
            if (base + kStage >= n) break;  // last batch: no barrier
            if (__syncthreads_count(done ? 1 : 0) == G::kThreads) break;
        }
    }

    if (inside) {
        const size_t P = static_cast<size_t>(a.W) * a.H;
        const size_t pix = static_cast<size_t>(py) * a.W + px;
#pragma unroll
        for (int c = 0; c < C; ++c)
            a.layers[(static_cast<size_t>(lplane) * C + c) * P + pix] = acc[c];
        if (a.t_final) a.t_final[static_cast<size_t>(lplane) * P + pix] = T;
        if constexpr (AUX) {
            a.n_contrib[static_cast<size_t>(lplane) * P + pix] = contrib;
            if (a.e_last) a.e_last[static_cast<size_t>(lplane) * P + pix] = elast;
        }
    }
}

// 16x16 tiles, PPT (2 or 4) pixels per thread: 256 / PPT threads, each warp an
// 8 x 4 PPT block, each lane the pixels (x, y + 4 k), k < PPT.  A hit entry's staged
// record is read once for all of a lane's pixels, and the quadratic forms of pixel
// pairs are evaluated with packed fp32x2 arithmetic; every packed operation rounds
// per element exactly as the scalar one of eval_alpha, so each pixel's alpha --
// hence every accept decision -- is the one k_composite, the backward and the
// brute force compute.
template <int C, bool AUX, int PPT>
__global__ void __launch_bounds__(256 / PPT, PPT == 2 ? HOLO_COMP2_MINB : HOLO_COMP4_MINB) k_composite2(CompositeArgs a) {
    constexpr int TILE = 16, NT = 256 / PPT;
    constexpr int kUnroll = HOLO_COMP2_UNROLL;
    constexpr int kStage = 256;
    constexpr int kTest = HOLO_COMP_TEST;
    static_assert(PPT % 2 == 0, "pixels are evaluated in pairs");
    union Smem {
        struct {
            unsigned long long key[kSortCap];
            int gid[kSortCap];
        } sort;
        struct {
            Staged rec[kStage + 1];
            float4 box[kStage];
        } st;
    };
    __shared__ Smem sm;
    __shared__ int s_ord[kSortCap];
    __shared__ __align__(8) int s_hit[NT / 32][32 * kTest + 2];

    const int tx = blockIdx.x, ty = blockIdx.y, lplane = blockIdx.z;
    const int lb = (lplane * gridDim.y + ty) * gridDim.x + tx;
    const int px0 = tx * TILE, py0 = ty * TILE;
    const unsigned e0 = min(a.bstart[lb], a.capacity);
    const int n = static_cast<int>(min(a.bstart[lb + 1], a.capacity) - e0);
    const int plane = a.plane_begin + lplane;

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int bx = (warp & 1) * 8, by = (warp >> 1) * (4 * PPT);
    const int lx = bx + (lane & 7), ly = by + (lane >> 3);  // pixels (lx, ly + 4 k)
    const int px = px0 + lx, py = py0 + ly;
    const float eps = a.term_eps;

    bool in[PPT];
    float T[PPT];
    int contrib[PPT], elast[PPT];
    cx<float> acc[PPT][C];
    bool done = true;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        in[k] = px < a.W && py + 4 * k < a.H;
        T[k] = 1.0f;
        contrib[k] = 0;
        elast[k] = -1;
#pragma unroll
        for (int c = 0; c < C; ++c) acc[k][c] = mk(0.0f, 0.0f);
        done = done && !(in[k] && 1.0f >= eps);
    }

    if (n > 0) {
        const bool presorted = n <= kWarpSortCap || n > kSortCap;
        if (!presorted) sort_bucket_cta<NT>(a, e0, n, tid, sm.sort.key, sm.sort.gid, s_ord);

        const float fx = static_cast<float>(lx) + 0.5f;
        unsigned long long fy2[PPT / 2];
#pragma unroll
        for (int j = 0; j < PPT / 2; ++j)
            fy2[j] = f32x2::pack(static_cast<float>(ly + 8 * j) + 0.5f, static_cast<float>(ly + 8 * j + 4) + 0.5f);
        const float bxlo = static_cast<float>(bx) + 0.5f, bxhi = static_cast<float>(bx) + 7.5f;
        const float bylo = static_cast<float>(by) + 0.5f, byhi = static_cast<float>(by + 4 * PPT - 1) + 0.5f;
        const float thr = a.floor_positive ? a.alpha_floor : 0.0f;
        const float clamp = a.alpha_clamp;
        // a pixel outside the image is parked with T = -1: never accepts, never written
#pragma unroll
        for (int k = 0; k < PPT; ++k)
            if (!in[k]) T[k] = -1.0f;

        for (int base = 0; base < n; base += kStage) {
            const int cnt = (n - base) < kStage ? (n - base) : kStage;
            for (int t = tid; t < cnt; t += NT) {
                const int g = presorted ? a.egidx[e0 + base + t] : s_ord[base + t];
                const GRec r = a.rec[g];
                float alpha = r.alpha;
                if (a.soft)
                    alpha = static_cast<float>(static_cast<double>(r.alpha) * a.rho[static_cast<size_t>(g) * a.L + plane]);
                stage_entry(r, px0, py0, alpha, sm.st.rec[t], sm.st.box[t]);
            }
            if (tid == 0) {
                Staged& z = sm.st.rec[kStage];
                z.a = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                z.b = make_float4(0.0f, -INFINITY, 0.0f, 0.0f);
                z.c = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            }
            __syncthreads();
            if (!__all_sync(0xffffffffu, done)) {
                // hits[] holds shared-window addresses: the walk's loads use them as is
                const unsigned recs = static_cast<unsigned>(__cvta_generic_to_shared(sm.st.rec));
                int* hits = s_hit[warp];
                for (int c0 = 0; c0 < cnt; c0 += 32 * kTest) {
                    const unsigned below = (1u << lane) - 1u;
                    int nh = 0;
#pragma unroll
                    for (int q = 0; q < kTest; ++q) {
                        const int j = c0 + 32 * q + lane;
                        const bool h = j < cnt && box_hits(sm.st.box[j], bxlo, bxhi, bylo, byhi);
                        const unsigned m = __ballot_sync(0xffffffffu, h);
                        if (h) hits[nh + __popc(m & below)] = static_cast<int>(recs + j * sizeof(Staged));
                        nh += __popc(m);
                    }
                    __syncwarp();
#ifdef HOLO_COUNT
                    unsigned long long n_any = 0;
#endif
#pragma unroll(kUnroll)
                    for (int kh = 0; kh < nh; ++kh) {
                        const unsigned ad = static_cast<unsigned>(hits[kh]);
                        const float4 A = lds128(ad), B = lds128(ad + 16);
                        const float4 Cc = C > 1 ? lds128(ad + 32) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                        // eval_alpha per pixel: d = centre - mu (dx shared), then
                        // t = fma(cb, dy, ca dx), u = fma(dx, t, log2 alpha),
                        // q = fma(cc dy, dy, u), a = min(2^q, clamp)
                        const float dx = fx - A.x;
                        const float cadx = A.z * dx;
                        const unsigned long long my2 = f32x2::pack(A.y, A.y), cb2 = f32x2::pack(A.w, A.w);
                        const unsigned long long cadx2 = f32x2::pack(cadx, cadx), dx2 = f32x2::pack(dx, dx);
                        const unsigned long long la2 = f32x2::pack(B.y, B.y), cc2 = f32x2::pack(B.x, B.x);
                        const int ei = base + static_cast<int>((ad - recs) / sizeof(Staged));
#pragma unroll
                        for (int j = 0; j < PPT / 2; ++j) {
                            const unsigned long long dy = f32x2::sub(fy2[j], my2);
                            const unsigned long long t = f32x2::fma(cb2, dy, cadx2);
                            const unsigned long long u = f32x2::fma(dx2, t, la2);
                            const cx<float> qq = f32x2::unpack(f32x2::fma(f32x2::mul(cc2, dy), dy, u));
                            const float al0 = fminf(ex2_approx(qq.x), clamp);
                            const float al1 = fminf(ex2_approx(qq.y), clamp);
                            float& Ta = T[2 * j];
                            float& Tb = T[2 * j + 1];
                            const cx<float> wt = f32x2::unpack(f32x2::mul(f32x2::pack(al0, al1), f32x2::pack(Ta, Tb)));
#if HOLO_COMP_PRED
                            // accept = (a > floor) and (T >= eps): one compare folds the other's
                            // predicate in, one select per pixel
                            const float w0 = accept_weight(al0, thr, Ta, eps, wt.x);
                            const float w1 = accept_weight(al1, thr, Tb, eps, wt.y);
                            const bool a0 = (al0 > thr) && (Ta >= eps);  // AUX only
                            const bool a1 = (al1 > thr) && (Tb >= eps);
#else
                            const bool a0 = (al0 > thr) && (Ta >= eps);
                            const bool a1 = (al1 > thr) && (Tb >= eps);
                            const float w0 = a0 ? wt.x : 0.0f, w1 = a1 ? wt.y : 0.0f;
#endif
                            blend_c<C>(B, Cc, w0, acc[2 * j]);
                            blend_c<C>(B, Cc, w1, acc[2 * j + 1]);
                            const cx<float> Tn = f32x2::unpack(f32x2::sub(f32x2::pack(Ta, Tb), f32x2::pack(w0, w1)));
                            Ta = Tn.x;
                            Tb = Tn.y;
                            if constexpr (AUX) {
                                contrib[2 * j] += a0 ? 1 : 0;
                                contrib[2 * j + 1] += a1 ? 1 : 0;
                                elast[2 * j] = a0 ? ei : elast[2 * j];
                                elast[2 * j + 1] = a1 ? ei : elast[2 * j + 1];
                            }
#ifdef HOLO_COUNT
                            n_any += __any_sync(0xffffffffu, (al0 > thr) || (al1 > thr)) ? 1 : 0;
#endif
                        }
                    }
#ifdef HOLO_COUNT
                    if (lane == 0) {
                        atomicAdd(&g_counts[0], static_cast<unsigned long long>(nh));
                        atomicAdd(&g_counts[1], n_any);
                    }
#endif
                    __syncwarp();
                    done = true;
#pragma unroll
                    for (int k = 0; k < PPT; ++k) done = done && !(T[k] >= eps);
                    if (__all_sync(0xffffffffu, done)) break;
                }
            }
            if (base + kStage >= n) break;
            if (__syncthreads_count(done ? 1 : 0) == NT) break;
        }
    }

    // outputs: one 64-bit base per array, then 32-bit steps of 4 rows / one channel
    const size_t P = static_cast<size_t>(a.W) * a.H;
    const size_t pix0 = static_cast<size_t>(lplane) * P + static_cast<size_t>(py) * a.W + px;
    cx<float>* lay = a.layers + static_cast<size_t>(lplane) * (C - 1) * P + pix0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        if (!in[k]) continue;
        const int dk = 4 * k * a.W;
#pragma unroll
        for (int c = 0; c < C; ++c) lay[static_cast<size_t>(c) * P + dk] = acc[k][c];
        if (a.t_final) a.t_final[pix0 + dk] = T[k];
        if constexpr (AUX) {
            a.n_contrib[pix0 + dk] = contrib[k];
            if (a.e_last) a.e_last[pix0 + dk] = elast[k];
        }
    }
}

#ifdef HOLO_COUNT
__global__ void k_print_counts() {
    printf("composite counts: warp-evals %llu, with any accept %llu, accepted lanes %llu, chunks %llu\n",
           g_counts[0], g_counts[1], g_counts[2], g_counts[3]);
    for (int i = 0; i < 4; ++i) g_counts[i] = 0;
}
#endif

template <int TILE>
void launch_tile(holo_ctx* ctx, const CompositeArgs& a) {
    if (a.num_buckets <= 0) return;
    const int tiles_y = a.num_tiles / a.tiles_x;
    const dim3 grid(a.tiles_x, tiles_y, a.num_buckets / a.num_tiles);
    if constexpr (TILE == 16) {
        if (HOLO_COMP2) {
            switch (a.C) {
#define HC_COMP2(CC)                                                                                          \
    (a.n_contrib ? k_composite2<CC, true, HOLO_COMP_PPT><<<grid, 256 / HOLO_COMP_PPT, 0, ctx->stream>>>(a)      \
                 : k_composite2<CC, false, HOLO_COMP_PPT><<<grid, 256 / HOLO_COMP_PPT, 0, ctx->stream>>>(a))
                case 1: HC_COMP2(1); break;
                case 2: HC_COMP2(2); break;
                case 3: HC_COMP2(3); break;
#undef HC_COMP2
                default: throw Error(HOLO_ERR_CONFIG, "render supports 1 to 3 wavelength channels");
            }
            HC_LAUNCHED(ctx);
#ifdef HOLO_COUNT
            k_print_counts<<<1, 1, 0, ctx->stream>>>();
#endif
            return;
        }
    }
    switch (a.C) {
#define HC_COMP(CC)                                                                   \
    (a.n_contrib ? k_composite<TILE, CC, true><<<grid, TILE * TILE, 0, ctx->stream>>>(a) \
                 : k_composite<TILE, CC, false><<<grid, TILE * TILE, 0, ctx->stream>>>(a))
        case 1: HC_COMP(1); break;
        case 2: HC_COMP(2); break;
        case 3: HC_COMP(3); break;
#undef HC_COMP
        default: throw Error(HOLO_ERR_CONFIG, "render supports 1 to 3 wavelength channels");
    }
    HC_LAUNCHED(ctx);
#ifdef HOLO_COUNT
    k_print_counts<<<1, 1, 0, ctx->stream>>>();
#endif
}

}  // namespace

void sort_small_buckets(holo_ctx* ctx, const unsigned* bstart, long long B, unsigned capacity,
                        const unsigned long long* zkey, int* egidx, unsigned* d_nlist) {
    if (B <= 0) return;
    const size_t max_large = capacity / (kSortCap + 1) + 1, max_mid = capacity / 129 + 1;
    int* large = static_cast<int*>(ctx->buffer("large_list", sizeof(int) * max_large));
    int* mid = static_cast<int*>(ctx->buffer("mid_list", sizeof(int) * max_mid));
    k_sort_small<<<static_cast<unsigned>((B + HOLO_SORT_SMALL_WARPS - 1) / HOLO_SORT_SMALL_WARPS), 32 * HOLO_SORT_SMALL_WARPS, 0,
                   ctx->stream>>>(
        bstart, B, capacity, zkey, egidx, large, static_cast<unsigned>(max_large), mid, static_cast<unsigned>(max_mid),
        d_nlist);
    HC_LAUNCHED(ctx);
}

void composite(holo_ctx* ctx, const CompositeArgs& a, int tile) {
    switch (tile) {
        case 8: launch_tile<8>(ctx, a); break;
        case 16: launch_tile<16>(ctx, a); break;
        case 32: launch_tile<32>(ctx, a); break;
        default: throw Error(HOLO_ERR_CONFIG, "render supports tile sizes 8, 16 and 32");
    }
}

}  // namespace holo_cuda
