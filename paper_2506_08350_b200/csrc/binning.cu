// Tile binning on sm_100a: (plane, tile) bucket histogram, exclusive scan into
// bucket_start, and emission of (depth key, Gaussian) work items.
//
// Replaces the serial emission / counting sort / per-bucket std::sort of
// raster_forward (proj/src/rasterizer.cpp:172-225).  Emission order inside a
// bucket is arbitrary here (atomic cursors); the compositing kernel restores the
// reference order by sorting each bucket on the total order (zc, gidx)
// (rasterizer.cpp:221-224), so the final lists are deterministic and equal the
// reference's.  Buckets above kSortCap entries are sorted here instead, by a
// single-CTA bitonic network per bucket.
#include <algorithm>

#include "kernels.cuh"
#include "sort_warp.cuh"

namespace holo_cuda {

namespace {

constexpr int kScanThreads = 256;
#ifndef HOLO_SCAN_ITEMS
#define HOLO_SCAN_ITEMS 4  // 1024-count tiles: C3 binning -4 us against 4096
#endif
constexpr int kScanItems = HOLO_SCAN_ITEMS;
constexpr int kScanTile = kScanThreads * kScanItems;
#ifndef HOLO_SCAN_ONEPASS
#define HOLO_SCAN_ONEPASS 1
#endif

__device__ __forceinline__ unsigned warp_incl_scan(unsigned v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned u = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += u;
    }
    return v;
}

// Exclusive block scan of one value per thread; returns the exclusive prefix, total in *total.
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* total) {
    __shared__ unsigned warp_sums[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const unsigned inc = warp_incl_scan(v);
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        unsigned s = lane < nw ? warp_sums[lane] : 0u;
        s = warp_incl_scan(s);
        if (lane < nw) warp_sums[lane] = s;
    }
    __syncthreads();
    const unsigned warp_prefix = wid > 0 ? warp_sums[wid - 1] : 0u;
    *total = warp_sums[nw - 1];
    __syncthreads();
    return warp_prefix + inc - v;
}

// the scanned sequence is in[i] + in2[i] (in2 may be null)
__global__ void __launch_bounds__(kScanThreads) k_scan_partials(const unsigned* __restrict__ in,
                                                                const unsigned* __restrict__ in2, long long n,
                                                                unsigned* __restrict__ partials,
                                                                unsigned* __restrict__ dmax) {
    const long long base = static_cast<long long>(blockIdx.x) * kScanTile;
    unsigned s = 0, m = 0;
    for (int k = 0; k < kScanItems; ++k) {
        const long long i = base + static_cast<long long>(k) * kScanThreads + threadIdx.x;
        if (i < n) {
            const unsigned v = in[i] + (in2 ? in2[i] : 0u);
            s += v;
            m = v > m ? v : m;
        }
    }
    unsigned total;
    block_excl_scan(s, &total);
    if (threadIdx.x == 0) partials[blockIdx.x] = total;
    // block max
    for (int d = 16; d > 0; d >>= 1) {
        const unsigned o = __shfl_down_sync(0xffffffffu, m, d);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0 && dmax) atomicMax(dmax, m);
}

__global__ void __launch_bounds__(kScanThreads) k_scan_top(unsigned* __restrict__ partials, int nblocks) {
    unsigned carry = 0;
    for (int base = 0; base < nblocks; base += kScanThreads) {
        const int i = base + threadIdx.x;
        const unsigned v = i < nblocks ? partials[i] : 0u;
        unsigned total;
        const unsigned ex = block_excl_scan(v, &total);
        if (i < nblocks) partials[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0) partials[nblocks] = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_final(const unsigned* __restrict__ in,
                                                             const unsigned* __restrict__ in2, long long n,
                                                             const unsigned* __restrict__ partials,
                                                             unsigned* __restrict__ out, int nblocks) {
    // each thread owns kScanItems consecutive elements
    const long long base = static_cast<long long>(blockIdx.x) * kScanTile + static_cast<long long>(threadIdx.x) * kScanItems;
    unsigned v[kScanItems];
    unsigned s = 0;
    for (int k = 0; k < kScanItems; ++k) {
        const long long i = base + k;
        v[k] = i < n ? in[i] + (in2 ? in2[i] : 0u) : 0u;
        s += v[k];
    }
    unsigned total;
    unsigned run = block_excl_scan(s, &total) + partials[blockIdx.x];
    for (int k = 0; k < kScanItems; ++k) {
        const long long i = base + k;
        if (i < n) out[i] = run;
        run += v[k];
    }
    if (blockIdx.x == nblocks - 1 && threadIdx.x == 0) out[n] = partials[nblocks];
}

// Single-pass exclusive scan with decoupled look-back: tiles are taken in launch
// order (an atomic ticket), each tile publishes its aggregate and then its
// inclusive prefix in a 64-bit status word (epoch:30 | flag:2 | value:32; flag 1 =
// aggregate, 2 = inclusive), and sums its predecessors' words until it meets an
// inclusive one.  The epoch (one per call) makes stale words of earlier calls
// invisible without clearing the array.  Integer sums: the result is exact and
// independent of the order.
__global__ void __launch_bounds__(kScanThreads) k_scan_onepass(const unsigned* __restrict__ in,
                                                              const unsigned* __restrict__ in2, long long n,
                                                              unsigned* __restrict__ out, unsigned* __restrict__ dmax,
                                                              unsigned long long* __restrict__ status,
                                                              unsigned* __restrict__ ticket, unsigned epoch,
                                                              unsigned ticket_base) {
    __shared__ unsigned s_tile, s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u) - ticket_base;
    __syncthreads();
    const int tile = static_cast<int>(s_tile);
    const long long base = static_cast<long long>(tile) * kScanTile + static_cast<long long>(threadIdx.x) * kScanItems;
    unsigned v[kScanItems];
    unsigned sum = 0, m = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const long long i = base + k;
        v[k] = i < n ? in[i] + (in2 ? in2[i] : 0u) : 0u;
        sum += v[k];
        m = v[k] > m ? v[k] : m;
    }
    unsigned total;
    const unsigned ex = block_excl_scan(sum, &total);
    const unsigned long long tag = static_cast<unsigned long long>(epoch & 0x3fffffffu) << 34;
    if (threadIdx.x < 32) {
        // warp-parallel look-back: 32 predecessors' status words per round trip,
        // summed up to the nearest one holding an inclusive prefix (flag 2); a
        // window with an unpublished word (flag 0) before that point is re-read
        const int lane = threadIdx.x;
        unsigned prefix = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&status[0], tag | (2ull << 32) | total);
        } else {
            if (lane == 0) atomicExch(&status[tile], tag | (1ull << 32) | total);
            for (int j = tile - 1; j >= 0;) {
                const int idx = j - lane;
                unsigned flag = 2, val = 0;  // before tile 0: an inclusive zero
                if (idx >= 0) {
                    const unsigned long long w = atomicAdd(&status[idx], 0ull);
                    flag = (w >> 34) != (tag >> 34) ? 0u : static_cast<unsigned>((w >> 32) & 3u);
                    val = static_cast<unsigned>(w);
                }
                const unsigned incl = __ballot_sync(0xffffffffu, flag == 2);
                const unsigned zero = __ballot_sync(0xffffffffu, flag == 0);
                const int stop = incl ? __ffs(incl) - 1 : 31;
                const unsigned upto = stop == 31 ? 0xffffffffu : (2u << stop) - 1u;
                if (zero & upto) continue;  // not yet published
                unsigned v = lane <= stop ? val : 0u;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
                prefix += v;
                if (incl) break;
                j -= 32;
            }
            if (lane == 0) atomicExch(&status[tile], tag | (2ull << 32) | (prefix + total));
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    unsigned run = s_prefix + ex;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const long long i = base + k;
        if (i < n) out[i] = run;
        run += v[k];
    }
    if (base <= n && n <= base + kScanItems) out[n] = run;  // the total, by the thread that ends at n
    if (dmax) {
        for (int d = 16; d > 0; d >>= 1) {
            const unsigned o = __shfl_down_sync(0xffffffffu, m, d);
            m = o > m ? o : m;
        }
        if ((threadIdx.x & 31) == 0) atomicMax(dmax, m);
    }
}

// Loop over the (plane, tile) buckets of Gaussian i restricted to planes [pb, pe).
template <class F>
__device__ __forceinline__ void for_each_bucket(const PreOut& pre, size_t i, int L, int pb, int pe, int tiles_x,
                                                int num_tiles, int soft, F f) {
    if (pre.count[i] == 0) return;
    const int4 r = pre.rect[i];
    if (soft) {
        const unsigned long long mask = pre.pmask[i];
        for (int l = pb; l < pe && l < 64; ++l) {
            if (!((mask >> l) & 1ull)) continue;
            for (int ty = r.z; ty < r.w; ++ty)
                for (int tx = r.x; tx < r.y; ++tx) f((l - pb) * num_tiles + ty * tiles_x + tx);
        }
    } else {
        const int l = pre.plane[i];
        if (l < pb || l >= pe) return;
        for (int ty = r.z; ty < r.w; ++ty)
            for (int tx = r.x; tx < r.y; ++tx) f((l - pb) * num_tiles + ty * tiles_x + tx);
    }
}

// (key, gidx) lexicographic order; zc > near > 0, so the IEEE bits of zc order like zc.
__device__ __forceinline__ bool less_kg(unsigned long long ka, int ga, unsigned long long kb, int gb) {
    return ka < kb || (ka == kb && ga < gb);
}

__global__ void __launch_bounds__(256) k_bucket_count(PreOut pre, size_t N, int L, int pb, int pe, int tiles_x,
                                                      int num_tiles, int soft, unsigned* __restrict__ bcount) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= N) return;
    for_each_bucket(pre, i, L, pb, pe, tiles_x, num_tiles, soft, [&](int b) { atomicAdd(bcount + b, 1u); });
}

#ifndef HOLO_EMIT_NT
#define HOLO_EMIT_NT 128  // measured: 256 0.0858, 128 0.0848, 64 0.0845 ms binning (C3)
#endif
__global__ void __launch_bounds__(HOLO_EMIT_NT) k_bucket_emit(PreOut pre, size_t N, int L, int pb, int pe, int tiles_x,
                                                     int num_tiles, int soft, const unsigned* __restrict__ bstart,
                                                     unsigned* __restrict__ cursor, int* __restrict__ egidx,
                                                     unsigned capacity, unsigned* __restrict__ flags) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= N) return;
    // every per-Gaussian load issued up front (one round trip instead of a chain)
    const unsigned cnt_i = pre.count[i];
    const int plane_i = soft ? 0 : pre.plane[i];
    const int4 rect_i = pre.rect[i];
    bool over = false;
    // entries beyond the reserved capacity (asynchronous frames) are dropped and flagged
    auto put = [&](int b, unsigned slot) {
        const unsigned e = bstart[b] + slot;
        if (e >= capacity) {
            over = true;
            return;
        }
        egidx[e] = static_cast<int>(i);
    };
    if (!soft) {
        if (cnt_i == 0) return;
        const int l = plane_i;
        if (l < pb || l >= pe) return;
        const int4 r = rect_i;
        const int w = r.y - r.x, n = w * (r.w - r.z);
        const int b0 = (l - pb) * num_tiles + r.z * tiles_x + r.x;
        if (pre.slots && n <= kSlots) {
            // slots taken in preprocess: no atomics; all slot and bucket-start
            // loads in flight before the first store
            // the k-th tile of the span, row-major: offsets stepped, no divisions
            unsigned st[kSlots];
            int off = 0, cx = 0;
#pragma unroll
            for (int k = 0; k < kSlots; ++k) {
                if (k < n) st[k] = bstart[b0 + off] + pre.slots[static_cast<size_t>(k) * N + i];
                ++off;
                if (++cx == w) {
                    cx = 0;
                    off += tiles_x - w;
                }
            }
#pragma unroll
            for (int k = 0; k < kSlots; ++k)
                if (k < n) {
                    const unsigned e = st[k];
                    if (e >= capacity) {
                        over = true;
                    } else {
                        egidx[e] = static_cast<int>(i);
                    }
                }
            if (over) atomicOr(flags, kFlagOverflow);
            return;
        }
        // the rect's tiles 4 at a time, so the slot atomics of a group are in flight
        // together instead of one round trip per entry; with preprocess slots, the
        // large Gaussians' slots follow the small ones' (bcount) in each bucket
        int off = 0, cx = 0;
        for (int k = 0; k < n; k += 4) {
            int b[4];
            unsigned s[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int idx = k + u;
                b[u] = b0 + off;
                ++off;
                if (++cx == w) {
                    cx = 0;
                    off += tiles_x - w;
                }
                if (idx < n) s[u] = atomicAdd(cursor + b[u], 1u) + (pre.slots ? pre.bcount[b[u]] : 0u);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k + u < n) put(b[u], s[u]);
        }
    } else {
        for_each_bucket(pre, i, L, pb, pe, tiles_x, num_tiles, soft,
                        [&](int b) { put(b, atomicAdd(cursor + b, 1u)); });
    }
    if (over) atomicOr(flags, kFlagOverflow);
}

// Persistent CTAs sort the listed buckets by (zc, gidx) with a bitonic network in
// global scratch; bucket b uses the scratch range [2 bstart[b], 2 bstart[b] + pow2(n)),
// which never overlaps another bucket's since pow2(n) < 2 n.
// The listed mid-size buckets come first, one warp each (eight keys per lane).
#ifndef HOLO_LARGE_NT
#define HOLO_LARGE_NT 256  // small CTAs: a frame without listed buckets does not hold whole SMs
#endif
#ifndef HOLO_LARGE_CTAS_PER_SM
#define HOLO_LARGE_CTAS_PER_SM 4
#endif
__global__ void __launch_bounds__(HOLO_LARGE_NT) k_sort_large_dev(const int* __restrict__ list,
                                                         const unsigned* __restrict__ nlist, unsigned max_list,
                                                         const int* __restrict__ mid, unsigned max_mid,
                                                         const unsigned* __restrict__ bstart, unsigned capacity,
                                                         const unsigned long long* __restrict__ zkey,
                                                         int* __restrict__ egidx,
                                                         unsigned long long* __restrict__ tkey, int* __restrict__ tg) {
    {
        const unsigned nmid = min(nlist[1], max_mid);
        const int lane = threadIdx.x & 31;
        // each CTA owns an equal contiguous range of the list; its warps take the
        // buckets one at a time from a shared-memory counter (a single global
        // counter serialised ~18 K same-address atomics at C4)
        __shared__ unsigned s_next;
        const unsigned per = (nmid + gridDim.x - 1) / gridDim.x;
        const unsigned lo = min(nmid, blockIdx.x * per), hi = min(nmid, lo + per);
        if (threadIdx.x == 0) s_next = lo;
        __syncthreads();
        while (true) {
            unsigned w = 0;
            if (lane == 0) w = atomicAdd(&s_next, 1u);
            w = __shfl_sync(0xffffffffu, w, 0);
            if (w >= hi) break;
            const int bk = mid[w];
            const unsigned e0 = min(bstart[bk], capacity);
            const int n = static_cast<int>(min(bstart[bk + 1], capacity) - e0);
            if (!warpsort::warp_sort_bucket_u32<8>(zkey, egidx, e0, n, lane) &&
                !warpsort::warp_sort_bucket_fast<8>(zkey, egidx, e0, n, lane))
                warpsort::warp_sort_bucket<8>(zkey, egidx, e0, n, lane);
        }
    }
    const unsigned count = min(*nlist, max_list);
    for (unsigned w = blockIdx.x; w < count; w += gridDim.x) {
        const int bk = list[w];
        const unsigned s = bstart[bk];
        unsigned n = bstart[bk + 1] - s;
        if (s >= capacity) continue;
        if (n > capacity - s) n = capacity - s;
        unsigned P = 1;
        while (P < n) P <<= 1;
        unsigned long long* K = tkey + 2 * static_cast<size_t>(s);
        int* G = tg + 2 * static_cast<size_t>(s);
        for (unsigned t = threadIdx.x; t < P; t += blockDim.x) {
            const int g = t < n ? egidx[s + t] : 0x7fffffff;
            K[t] = t < n ? zkey[g] : ~0ull;
            G[t] = g;
        }
        __syncthreads();
        for (unsigned k = 2; k <= P; k <<= 1) {
            for (unsigned j = k >> 1; j > 0; j >>= 1) {
                for (unsigned t = threadIdx.x; t < P; t += blockDim.x) {
                    const unsigned u = t ^ j;
                    if (u > t) {
                        const bool up = (t & k) == 0;
                        const unsigned long long ka = K[t], kb = K[u];
                        const int ga = G[t], gb = G[u];
                        const bool swap = up ? less_kg(kb, gb, ka, ga) : less_kg(ka, ga, kb, gb);
                        if (swap) {
                            K[t] = kb;
                            K[u] = ka;
                            G[t] = gb;
                            G[u] = ga;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (unsigned t = threadIdx.x; t < n; t += blockDim.x) egidx[s + t] = G[t];
        __syncthreads();
    }
}

// Entry::depth = zc[gidx] for e < min(E, capacity), E read on the device.
__global__ void k_entry_depths(const int* __restrict__ egidx, const double* __restrict__ zc,
                               double* __restrict__ edepth, const unsigned* __restrict__ d_E, unsigned capacity) {
    const unsigned E = *d_E < capacity ? *d_E : capacity;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < E;
         e += static_cast<size_t>(gridDim.x) * blockDim.x)
        edepth[e] = zc[egidx[e]];
}

}  // namespace

void exclusive_scan_u32(holo_ctx* ctx, const unsigned* in, unsigned* out, long long n, unsigned* d_max,
                        const unsigned* in2) {
    const int nblocks = static_cast<int>((n + kScanTile - 1) / kScanTile);
    const int nb = nblocks > 0 ? nblocks : 1;
    if (HOLO_SCAN_ONEPASS) {
        // The status words and the ticket persist across calls: each call takes a new
        // epoch (stale words of other calls never match it) and the ticket base it
        // starts from (every tile of a call takes one ticket).  Growth, epoch wrap and
        // ticket wrap start over on zeroed memory.
        holo_ctx::ScanState& stt = ctx->scan;
        auto* status = static_cast<unsigned long long*>(ctx->buffer("scan_status", sizeof(unsigned long long) * (nb + 64)));
        auto* ticket = reinterpret_cast<unsigned*>(status + nb + 32);
        if (nb > stt.cap || stt.epoch >= (1u << 30) - 1 ||
            static_cast<unsigned long long>(stt.ticket) + static_cast<unsigned>(nb) >= 0xffffffffull) {
            stt.cap = std::max(stt.cap, nb);
            status = static_cast<unsigned long long*>(ctx->buffer("scan_status", sizeof(unsigned long long) * (stt.cap + 64)));
            ticket = reinterpret_cast<unsigned*>(status + stt.cap + 32);
            HC_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * (stt.cap + 64), ctx->stream));
            stt.epoch = 1;
            stt.ticket = 0;
        }
        ticket = reinterpret_cast<unsigned*>(status + stt.cap + 32);
        k_scan_onepass<<<nb, kScanThreads, 0, ctx->stream>>>(in, in2, n, out, d_max, status, ticket, stt.epoch,
                                                             stt.ticket);
        HC_LAUNCHED(ctx);
        ++stt.epoch;
        stt.ticket += static_cast<unsigned>(nb);
        return;
    }
    unsigned* partials = static_cast<unsigned*>(ctx->buffer("scan_partials", sizeof(unsigned) * (nb + 1)));
    k_scan_partials<<<nb, kScanThreads, 0, ctx->stream>>>(in, in2, n, partials, d_max);
    HC_LAUNCHED(ctx);
    k_scan_top<<<1, kScanThreads, 0, ctx->stream>>>(partials, nb);
    HC_LAUNCHED(ctx);
    k_scan_final<<<nb, kScanThreads, 0, ctx->stream>>>(in, in2, n, partials, out, nb);
    HC_LAUNCHED(ctx);
}

void bucket_count(holo_ctx* ctx, const PreOut& pre, size_t N, int L, int pb, int pe, int tiles_x, int num_tiles,
                  int soft, unsigned* bcount) {
    if (N == 0) return;
    k_bucket_count<<<static_cast<unsigned>((N + 255) / 256), 256, 0, ctx->stream>>>(pre, N, L, pb, pe, tiles_x,
                                                                                    num_tiles, soft, bcount);
    HC_LAUNCHED(ctx);
}

void bucket_emit(holo_ctx* ctx, const PreOut& pre, size_t N, int L, int pb, int pe, int tiles_x, int num_tiles,
                 int soft, const unsigned* bstart, unsigned* cursor, int* egidx, unsigned capacity,
                 unsigned* flags) {
    if (N == 0) return;
    k_bucket_emit<<<static_cast<unsigned>((N + HOLO_EMIT_NT - 1) / HOLO_EMIT_NT), HOLO_EMIT_NT, 0, ctx->stream>>>(
        pre, N, L, pb, pe, tiles_x, num_tiles, soft, bstart, cursor, egidx, capacity, flags);
    HC_LAUNCHED(ctx);
}

void sort_large_buckets(holo_ctx* ctx, const unsigned* bstart, long long B, unsigned capacity,
                        const unsigned long long* zkey, int* egidx, unsigned* d_nlist) {
    // the lists k_sort_small built (sized as there)
    const size_t max_list = capacity / (kSortCap + 1) + 1, max_mid = capacity / 129 + 1;
    const int* list = static_cast<const int*>(ctx->buffer("large_list", sizeof(int) * max_list));
    const int* mid = static_cast<const int*>(ctx->buffer("mid_list", sizeof(int) * max_mid));
    auto* tkey = static_cast<unsigned long long*>(ctx->buffer("large_tkey", sizeof(unsigned long long) * 2 * (capacity + 1)));
    auto* tg = static_cast<int*>(ctx->buffer("large_tg", sizeof(int) * 2 * (capacity + 1)));
    // the lists are on the device: size the grid by the mean bucket (entry capacity
    // over buckets) -- one CTA per SM where listed buckets are unlikely, so an empty
    // pass costs the other frame in flight little
    const double mean = B > 0 ? static_cast<double>(capacity) / static_cast<double>(B) : 0.0;
    const int per_sm = mean > 96.0 ? HOLO_LARGE_CTAS_PER_SM : 1;
    k_sort_large_dev<<<ctx->sm_count * per_sm, HOLO_LARGE_NT, 0, ctx->stream>>>(list, d_nlist, static_cast<unsigned>(max_list), mid,
                                                             static_cast<unsigned>(max_mid), bstart, capacity, zkey,
                                                             egidx, tkey, tg);
    HC_LAUNCHED(ctx);
}

void entry_depths(holo_ctx* ctx, const int* egidx, const double* zc, double* edepth, const unsigned* d_E,
                  unsigned capacity) {
    if (capacity == 0) return;
    const size_t blocks = (static_cast<size_t>(capacity) + 255) / 256;
    const unsigned grid = static_cast<unsigned>(blocks < 4096 ? blocks : 4096);
    k_entry_depths<<<grid, 256, 0, ctx->stream>>>(egidx, zc, edepth, d_E, capacity);
    HC_LAUNCHED(ctx);
}

namespace {
// status words -> pinned host memory, stored by the SMs: no copy-engine transfer,
// which would queue behind the large downloads of earlier frames
__global__ void k_publish_status(const unsigned* __restrict__ misc, const unsigned* __restrict__ total,
                                 volatile unsigned* host) {
    const int t = threadIdx.x;
    if (t < 3) host[t] = misc[t];
    if (t == 4) host[4] = *total;
}
}  // namespace

void publish_status(holo_ctx* ctx, const unsigned* misc, const unsigned* total, unsigned* host_pinned) {
    k_publish_status<<<1, 32, 0, ctx->stream>>>(misc, total, host_pinned);
    HC_LAUNCHED(ctx);
}

}  // namespace holo_cuda
