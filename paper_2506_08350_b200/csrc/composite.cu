// K7 composite: per-(plane, tile) front-to-back complex alpha compositing (sm_100a).
//
// Restates the hot loop of raster_forward (proj/src/rasterizer.cpp:227-261) with
// evaluate() (:124-135): per pixel centre (px + 0.5, py + 0.5), in bucket order,
//   stop once T < term_eps (checked before each entry),
//   a = min(alpha * exp(-form / 2) * rho, alpha_clamp), skip unless a > alpha_floor,
//   acc_c += a T amp_c e^{i phi_c},  T *= 1 - a,  ++n_contrib.
// One CTA per bucket, one thread per pixel.  The CTA first restores the
// reference order of its bucket -- ascending (zc, gidx), rasterizer.cpp:221-224 --
// by a warp-shuffle bitonic sort (<= 128 entries), a rank sort (<= 256) or a
// shared-memory bitonic sort (<= kSortCap); larger buckets arrive presorted from
// binning.cu.  Records are staged 256 at a time in shared memory; each warp
// covers an 8x4 pixel block and, 32 entries per ballot, skips entries whose
// accept ellipse (a > alpha_floor) has a bounding box missing the block.  Evaluation is fp32 with the
// centre offset formed in f64 per entry, so dx, dy keep full fp32 precision.
#include "kernels.cuh"

namespace holo_cuda {

namespace {

// 2^x on the MUFU pipe (max rel. error 2^-22.5); x <= 0 here, results below 2^-126 flush to 0.
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int TILE>
struct TileGeom {
    static constexpr int kThreads = TILE * TILE;
    // warp block: 8 wide x 4 tall (TILE >= 8); TILE/8 blocks per row
    static constexpr int kBlocksX = TILE / 8;
};

struct KeyG {
    unsigned long long k;  // IEEE bits of zc (> 0, so they order like zc)
    int g;                 // Gaussian index: the tie-break
};

__device__ __forceinline__ bool kg_less(const KeyG& a, const KeyG& b) {
    return a.k < b.k || (a.k == b.k && a.g < b.g);
}

// Bitonic sort of 32 * NE (key, gidx) pairs held by one warp, element i in lane
// i % 32, slot i / 32; ascending on (zc, gidx) -- rasterizer.cpp:221-224.
template <int NE>
__device__ __forceinline__ void warp_bitonic(KeyG (&v)[NE], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * NE; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
#pragma unroll
                for (int s = 0; s < NE; ++s) {
                    const int s2 = s ^ (j >> 5);
                    if (s2 > s) {
                        const bool up = ((lane + 32 * s) & k) == 0;
                        const bool swap = up ? kg_less(v[s2], v[s]) : kg_less(v[s], v[s2]);
                        if (swap) {
                            const KeyG t = v[s];
                            v[s] = v[s2];
                            v[s2] = t;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int s = 0; s < NE; ++s) {
                    KeyG o;
                    o.k = __shfl_xor_sync(0xffffffffu, v[s].k, j);
                    o.g = __shfl_xor_sync(0xffffffffu, v[s].g, j);
                    const bool lower = (lane & j) == 0;
                    const bool up = ((lane + 32 * s) & k) == 0;
                    const bool take_min = lower == up;
                    const bool o_less = kg_less(o, v[s]);
                    if (take_min ? o_less : !o_less) v[s] = o;
                }
            }
        }
    }
}

// Sort one bucket (n <= 32 NE entries) in a warp.  PACK: the tie-break key carries
// the emission slot in its low 7 bits ((gidx << 7) | slot, n <= 128, gidx < 2^24),
// which orders exactly like gidx, and s_ord receives slots instead of indices.
template <int NE, bool PACK>
__device__ __forceinline__ void warp_sort_bucket(const unsigned long long* __restrict__ ekey,
                                                 const int* __restrict__ egidx, unsigned e0, int n, int lane,
                                                 int* __restrict__ s_ord) {
    KeyG v[NE];
#pragma unroll
    for (int s = 0; s < NE; ++s) {
        const int i = lane + 32 * s;
        v[s].k = i < n ? ekey[e0 + i] : ~0ull;
        v[s].g = i < n ? (PACK ? ((egidx[e0 + i] << 7) | i) : egidx[e0 + i]) : 0x7fffffff;
    }
    warp_bitonic<NE>(v, lane);
#pragma unroll
    for (int s = 0; s < NE; ++s) {
        const int i = lane + 32 * s;
        if (i < n) s_ord[i] = PACK ? (v[s].g & 127) : v[s].g;
    }
}

template <int NE, bool PACK>
__device__ __forceinline__ void warp_sort_any(const CompositeArgs& a, unsigned e0, int n, int lane, int* s_ord) {
    if (n <= 32)
        warp_sort_bucket<1, PACK>(a.ekey, a.egidx, e0, n, lane, s_ord);
    else if (n <= 64)
        warp_sort_bucket<2, PACK>(a.ekey, a.egidx, e0, n, lane, s_ord);
    else
        warp_sort_bucket<4, PACK>(a.ekey, a.egidx, e0, n, lane, s_ord);
}

// One staged entry: 64 bytes, read with four 16-byte shared loads from one base.
struct alignas(16) Staged {
    float4 a;  // mx, my, ca, cb   (centre relative to the tile origin; conic, log2-scaled)
    float4 b;  // cc, alpha, ylo, yhi
    float4 c;  // xlo, xhi, col0 re, col0 im
    float4 d;  // col1 re, col1 im, col2 re, col2 im
};

template <int TILE, int C>
__global__ void __launch_bounds__(TILE * TILE) k_composite(CompositeArgs a) {
    using G = TileGeom<TILE>;
    __shared__ unsigned long long s_key[kSortCap];
    __shared__ int s_gid[kSortCap];
    __shared__ int s_ord[kSortCap];
    constexpr int kStage = 256;  // records staged per batch
    __shared__ Staged s_rec[kStage];

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

    float T = 1.0f;
    int contrib = 0;
    float acc[2 * C];
#pragma unroll
    for (int c = 0; c < 2 * C; ++c) acc[c] = 0.0f;
    bool done = !inside || !(1.0f >= a.term_eps);  // the reference checks T < term_eps before every entry

    if (n > 0) {
        // ---- restore the reference order (zc asc, gidx asc): warp-shuffle bitonic
        // for <= 128 entries, rank / shared bitonic sorts up to kSortCap, presorted
        // by binning.cu beyond
        const bool presorted = n > kSortCap;
        if (!presorted) {
            if (n <= 128) {
                if (warp == 0) warp_sort_any<4, false>(a, e0, n, lane, s_ord);
            } else {
                for (int t = tid; t < n; t += G::kThreads) {
                    s_key[t] = a.ekey[e0 + t];
                    s_gid[t] = a.egidx[e0 + t];
                }
                __syncthreads();
                if (n <= G::kThreads) {
                    if (tid < n) {
                        const unsigned long long k = s_key[tid];
                        const int g = s_gid[tid];
                        int rank = 0;
                        for (int j = 0; j < n; ++j) {
                            const unsigned long long kj = s_key[j];
                            rank += (kj < k || (kj == k && s_gid[j] < g)) ? 1 : 0;
                        }
                        s_ord[rank] = g;
                    }
                } else {
                    int P = 1;
                    while (P < n) P <<= 1;
                    for (int t = n + tid; t < P; t += G::kThreads) {
                        s_key[t] = ~0ull;
                        s_gid[t] = 0x7fffffff;
                    }
                    __syncthreads();
                    for (int k = 2; k <= P; k <<= 1) {
                        for (int j = k >> 1; j > 0; j >>= 1) {
                            for (int t = tid; t < P; t += G::kThreads) {
                                const int u = t ^ j;
                                if (u > t) {
                                    const bool up = (t & k) == 0;
                                    const unsigned long long ka = s_key[t], kb = s_key[u];
                                    const int ga = s_gid[t], gb = s_gid[u];
                                    const bool b_less = kb < ka || (kb == ka && gb < ga);
                                    const bool a_less = ka < kb || (ka == kb && ga < gb);
                                    if (up ? b_less : a_less) {
                                        s_key[t] = kb;
                                        s_key[u] = ka;
                                        s_gid[t] = gb;
                                        s_gid[u] = ga;
                                    }
                                }
                            }
                            __syncthreads();
                        }
                    }
                    for (int t = tid; t < n; t += G::kThreads) s_ord[t] = s_gid[t];
                }
            }
            __syncthreads();
            if (a.write_lists)
                for (int t = tid; t < n; t += G::kThreads) a.egidx[e0 + t] = s_ord[t];
        }

        const float fx = static_cast<float>(lx) + 0.5f, fy = static_cast<float>(ly) + 0.5f;
        const float bxlo = static_cast<float>(bx) + 0.5f, bxhi = static_cast<float>(bx) + 7.5f;
        const float bylo = static_cast<float>(by) + 0.5f, byhi = static_cast<float>(by) + 3.5f;
        // accept = a > alpha_floor, or a > 0 without a positive floor (rasterizer.cpp:133)
        const float thr = a.floor_positive ? a.alpha_floor : 0.0f;

        for (int base = 0; base < n; base += kStage) {
            const int cnt = (n - base) < kStage ? (n - base) : kStage;
            // stage sorted records: tile-relative centre (formed in f64), conic, alpha
            // (times rho in soft mode), accept-ellipse box, channel phasors
            for (int t = tid; t < cnt; t += G::kThreads) {
                const int g = presorted ? a.egidx[e0 + base + t] : s_ord[base + t];
                const GRec r = a.rec[g];
                const float mx = static_cast<float>(r.mu_x - static_cast<double>(px0));
                const float my = static_cast<float>(r.mu_y - static_cast<double>(py0));
                float alpha = r.alpha;
                if (a.soft)
                    alpha = static_cast<float>(static_cast<double>(r.alpha) * a.rho[static_cast<size_t>(g) * a.L + plane]);
                Staged st;
                st.a = make_float4(mx, my, r.ca, r.cb);
                st.b = make_float4(r.cc, alpha, my - r.hy, my + r.hy);
                st.c = make_float4(mx - r.hx, mx + r.hx, r.col[0], r.col[1]);
                st.d = make_float4(r.col[2], r.col[3], r.col[4], r.col[5]);
                s_rec[t] = st;
            }
            __syncthreads();
            if (!__all_sync(0xffffffffu, done)) {
                // 32 entries at a time: each lane tests one entry's accept box against
                // this warp's 8x4 block of pixel centres; the warp walks the hits in
                // order, branch-free per lane (predicated accept).
                for (int c0 = 0; c0 < cnt; c0 += 32) {
                    bool hit = false;
                    if (c0 + lane < cnt) {
                        const float4 Bb = s_rec[c0 + lane].b;
                        const float4 Cb = s_rec[c0 + lane].c;
                        hit = !(Cb.y < bxlo || Cb.x > bxhi || Bb.w < bylo || Bb.z > byhi);
                    }
                    unsigned mask = __ballot_sync(0xffffffffu, hit);
                    while (mask) {
                        const Staged* e = &s_rec[c0 + __ffs(mask) - 1];
                        mask &= mask - 1;
                        const float4 A = e->a;
                        const float4 B = e->b;
                        const float dx = fx - A.x, dy = fy - A.y;
                        const float q = dx * fmaf(A.z, dx, A.w * dy) + B.x * dy * dy;
                        const float al = fminf(B.y * ex2_approx(q), a.alpha_clamp);
                        const bool accept = (al > thr) && !done;
                        const float w = accept ? al * T : 0.0f;
                        const float4 Cc = e->c;
                        acc[0] = fmaf(w, Cc.z, acc[0]);
                        acc[1] = fmaf(w, Cc.w, acc[1]);
                        if (C > 1) {
                            const float4 D = e->d;
                            acc[2 % (2 * C)] = fmaf(w, D.x, acc[2 % (2 * C)]);
                            acc[3 % (2 * C)] = fmaf(w, D.y, acc[3 % (2 * C)]);
                            if (C > 2) {
                                acc[4 % (2 * C)] = fmaf(w, D.z, acc[4 % (2 * C)]);
                                acc[5 % (2 * C)] = fmaf(w, D.w, acc[5 % (2 * C)]);
                            }
                        }
                        T -= w;  // T (1 - a)
                        contrib += accept ? 1 : 0;
                        done = done || (T < a.term_eps);
                    }
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
            a.layers[(static_cast<size_t>(lplane) * C + c) * P + pix] = mk(acc[2 * c], acc[2 * c + 1]);
        if (a.t_final) a.t_final[static_cast<size_t>(lplane) * P + pix] = T;
        if (a.n_contrib) a.n_contrib[static_cast<size_t>(lplane) * P + pix] = contrib;
    }
}

template <int TILE>
void launch_tile(holo_ctx* ctx, const CompositeArgs& a) {
    if (a.num_buckets <= 0) return;
    const int tiles_y = a.num_tiles / a.tiles_x;
    const dim3 grid(a.tiles_x, tiles_y, a.num_buckets / a.num_tiles);
    switch (a.C) {
        case 1: k_composite<TILE, 1><<<grid, TILE * TILE, 0, ctx->stream>>>(a); break;
        case 2: k_composite<TILE, 2><<<grid, TILE * TILE, 0, ctx->stream>>>(a); break;
        case 3: k_composite<TILE, 3><<<grid, TILE * TILE, 0, ctx->stream>>>(a); break;
        default: throw Error(HOLO_ERR_CONFIG, "render supports 1 to 3 wavelength channels");
    }
    HC_LAUNCHED(ctx);
}

}  // namespace

void composite(holo_ctx* ctx, const CompositeArgs& a, int tile) {
    switch (tile) {
        case 8: launch_tile<8>(ctx, a); break;
        case 16: launch_tile<16>(ctx, a); break;
        case 32: launch_tile<32>(ctx, a); break;
        default: throw Error(HOLO_ERR_CONFIG, "render supports tile sizes 8, 16 and 32");
    }
}

}  // namespace holo_cuda
