// Warp-level bitonic sorts of one bucket's entries on the total order (zc, gidx)
// (rasterizer.cpp:221-224), shared by the small-bucket kernel (composite.cu) and
// the device-side mid / large bucket pass (binning.cu).
#pragma once

#include "kernels.cuh"

namespace holo_cuda {
namespace warpsort {

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

// Sort one bucket (n <= 32 NE entries) in a warp and write its gidx back in order.
template <int NE>
__device__ __forceinline__ void warp_sort_bucket(const unsigned long long* __restrict__ zkey, int* __restrict__ egidx,
                                                 unsigned e0, int n, int lane) {
    KeyG v[NE];
#pragma unroll
    for (int s = 0; s < NE; ++s) {
        const int i = lane + 32 * s;
        v[s].g = i < n ? egidx[e0 + i] : 0x7fffffff;
    }
#pragma unroll
    for (int s = 0; s < NE; ++s) v[s].k = lane + 32 * s < n ? zkey[v[s].g] : ~0ull;
    warp_bitonic<NE>(v, lane);
#pragma unroll
    for (int s = 0; s < NE; ++s) {
        const int i = lane + 32 * s;
        if (i < n) egidx[e0 + i] = v[s].g;
    }
}

// Bitonic sort of 32 * NE 64-bit keys held by one warp (layout as warp_bitonic).
template <int NE>
__device__ __forceinline__ void warp_bitonic_u64(unsigned long long (&v)[NE], int lane) {
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
                        const unsigned long long a = v[s], b = v[s2];
                        v[s] = up ? min(a, b) : max(a, b);
                        v[s2] = up ? max(a, b) : min(a, b);
                    }
                }
            } else {
#pragma unroll
                for (int s = 0; s < NE; ++s) {
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[s], j);
                    const bool lower = (lane & j) == 0;
                    const bool up = ((lane + 32 * s) & k) == 0;
                    v[s] = (lower == up) ? min(v[s], o) : max(v[s], o);
                }
            }
        }
    }
}

// Fast path of warp_sort_bucket: one 64-bit key per entry, (fp32 depth bits << 32 |
// gidx).  Rounding to fp32 is monotonic, so this order equals (zc, gidx) unless two
// entries share an fp32 depth with different f64 depths; that (rare) case is
// detected on the sorted sequence and the exact sort runs instead.  Returns false then.
template <int NE>
__device__ __forceinline__ bool warp_sort_bucket_fast(const unsigned long long* __restrict__ zkey,
                                                      int* __restrict__ egidx, unsigned e0, int n, int lane) {
    unsigned long long v[NE];
#pragma unroll
    for (int s = 0; s < NE; ++s) {
        const int i = lane + 32 * s;
        v[s] = i < n ? static_cast<unsigned long long>(static_cast<unsigned>(egidx[e0 + i])) : ~0ull;
    }
#pragma unroll
    for (int s = 0; s < NE; ++s)
        if (lane + 32 * s < n) {
            const float z = __double2float_rn(__longlong_as_double(static_cast<long long>(zkey[v[s]])));
            v[s] |= static_cast<unsigned long long>(__float_as_uint(z)) << 32;
        }
    warp_bitonic_u64<NE>(v, lane);
    bool tie = false;
#pragma unroll
    for (int s = 0; s < NE; ++s) {
        const unsigned long long dn = __shfl_down_sync(0xffffffffu, v[s], 1);
        const unsigned long long wrap = __shfl_sync(0xffffffffu, v[(s + 1) % NE], 0);
        const unsigned long long next = lane < 31 ? dn : wrap;
        const int i = lane + 32 * s;
        tie = tie || (i + 1 < n && (v[s] >> 32) == (next >> 32));
    }
    if (__any_sync(0xffffffffu, tie)) return false;
#pragma unroll
    for (int s = 0; s < NE; ++s) {
        const int i = lane + 32 * s;
        if (i < n) egidx[e0 + i] = static_cast<int>(v[s] & 0xffffffffull);
    }
    return true;
}

// Bitonic sort of 32 * NE 32-bit keys held by one warp (layout as warp_bitonic).
template <int NE>
__device__ __forceinline__ void warp_bitonic_u32(unsigned (&v)[NE], int lane) {
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
                        const unsigned a = v[s], b = v[s2];
                        v[s] = up ? min(a, b) : max(a, b);
                        v[s2] = up ? max(a, b) : min(a, b);
                    }
                }
            } else {
#pragma unroll
                for (int s = 0; s < NE; ++s) {
                    const unsigned o = __shfl_xor_sync(0xffffffffu, v[s], j);
                    const bool lower = (lane & j) == 0;
                    const bool up = ((lane + 32 * s) & k) == 0;
                    v[s] = (lower == up) ? min(v[s], o) : max(v[s], o);
                }
            }
        }
    }
}

// Fastest path: one 32-bit key per entry, (fp32 depth bits with the low SB - 1
// mantissa bits dropped) << SB | the entry's position in the bucket, SB = log2(32 NE).
// The truncated depth is monotonic in zc, so when no two entries share it this
// order is the (zc, gidx) order; a shared value is detected on the sorted sequence
// and the caller falls back to the 64-bit key (returns false).  Half the shuffles
// and a third of the compare-select work of the 64-bit key.
template <int NE>
__device__ __forceinline__ bool warp_sort_bucket_u32(const unsigned long long* __restrict__ zkey,
                                                     int* __restrict__ egidx, unsigned e0, int n, int lane) {
    constexpr int SB = NE == 1 ? 5 : NE == 2 ? 6 : NE == 4 ? 7 : 8;
    static_assert(32 * NE == (1 << SB), "one position per key slot");
    int gid[NE];
    unsigned v[NE];
#pragma unroll
    for (int s = 0; s < NE; ++s) {
        const int i = lane + 32 * s;
        gid[s] = i < n ? egidx[e0 + i] : 0;
    }
    if constexpr (NE < 8) {
#pragma unroll
        for (int s = 0; s < NE; ++s) {
            const int i = lane + 32 * s;
            v[s] = ~0u;
            if (i < n) {
                const float z = __double2float_rn(__longlong_as_double(static_cast<long long>(zkey[gid[s]])));
                v[s] = ((__float_as_uint(z) >> (SB - 1)) << SB) | static_cast<unsigned>(i);
            }
        }
    } else {
        // 129..256 entries: 24 bits of truncated depth would collide in most
        // buckets (birthday bound), so the depth is quantised over the bucket's own
        // range instead, q = (z - zmin) (2^24 - 1) / (zmax - zmin) -- every step
        // monotonic, so distinct q still give the (zc, gidx) order
        constexpr unsigned kQMax = (1u << (32 - SB)) - 1u;
        float z[NE];
        float zlo = INFINITY, zhi = -INFINITY;
#pragma unroll
        for (int s = 0; s < NE; ++s) {
            const int i = lane + 32 * s;
            z[s] = 0.0f;
            if (i < n) {
                z[s] = __double2float_rn(__longlong_as_double(static_cast<long long>(zkey[gid[s]])));
                zlo = fminf(zlo, z[s]);
                zhi = fmaxf(zhi, z[s]);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            zlo = fminf(zlo, __shfl_xor_sync(0xffffffffu, zlo, o));
            zhi = fmaxf(zhi, __shfl_xor_sync(0xffffffffu, zhi, o));
        }
        if (!(zhi > zlo)) return false;  // one fp32 depth for all: the 64-bit key decides
        const float scale = static_cast<float>(kQMax) / (zhi - zlo);
#pragma unroll
        for (int s = 0; s < NE; ++s) {
            const int i = lane + 32 * s;
            v[s] = ~0u;
            if (i < n) v[s] = (min(__float2uint_rz((z[s] - zlo) * scale), kQMax) << SB) | static_cast<unsigned>(i);
        }
    }
    warp_bitonic_u32<NE>(v, lane);
    bool tie = false;
#pragma unroll
    for (int s = 0; s < NE; ++s) {
        const unsigned dn = __shfl_down_sync(0xffffffffu, v[s], 1);
        const unsigned wrap = __shfl_sync(0xffffffffu, v[(s + 1) % NE], 0);
        const unsigned next = lane < 31 ? dn : wrap;
        const int i = lane + 32 * s;
        tie = tie || (i + 1 < n && (v[s] >> SB) == (next >> SB));
    }
    if (__any_sync(0xffffffffu, tie)) return false;
#pragma unroll
    for (int s = 0; s < NE; ++s) {
        const int src = static_cast<int>(v[s] & ((1u << SB) - 1));
        int g = 0;
#pragma unroll
        for (int u = 0; u < NE; ++u) {
            const int gu = __shfl_sync(0xffffffffu, gid[u], src & 31);
            if ((src >> 5) == u) g = gu;
        }
        const int i = lane + 32 * s;
        if (i < n) egidx[e0 + i] = g;
    }
    return true;
}

}  // namespace warpsort
}  // namespace holo_cuda
