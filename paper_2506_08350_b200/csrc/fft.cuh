// Mixed-radix Stockham FFT building blocks for sm_100a.
//
// Replaces FFTW's c2c 2-D transform (reference proj/src/fft.cpp:33-44) with
// batched 1-D passes over shared-memory tiles.  Convention (fft.hpp:7-10):
// forward exp(-2 pi i jk/n) unnormalised, inverse exp(+2 pi i jk/n); the caller
// applies the 1/(w h) of ifft2 in its epilogue.
//
// A length-n transform is a sequence of self-sorting Stockham stages with radices
// from {2..16} and primes up to 31.  Each butterfly is an in-register DFT codelet
// (compile-time constants from fft_consts.cuh); the inter-stage twiddles come
// from a table exp(-2 pi i q / n), q < n, computed in double on the host.
#pragma once

#include "common.cuh"
#include "fft_consts.cuh"

#include <cstring>
#include <vector>

namespace holo_cuda {

constexpr int kMaxStages = 16;

struct FftPlan {
    int n;
    int nstages;
    int radix[kMaxStages];
};

// Host: factor n into Stockham radices; false if a prime factor exceeds 31.
// 3s pair with 5s (15) then with each other (9); 2s go in 16s, a remainder
// merges with a lone 3 (6, 12) or 5 (10); other primes <= 31 stay alone.
inline bool make_plan(int n, FftPlan* p) {
    std::memset(p, 0, sizeof *p);
    p->n = n;
    if (n < 1) return false;
    int e2 = 0, e3 = 0, e5 = 0;
    int m = n;
    while (m % 2 == 0) { m /= 2; ++e2; }
    while (m % 3 == 0) { m /= 3; ++e3; }
    while (m % 5 == 0) { m /= 5; ++e5; }
    std::vector<int> rad;
    for (int q : {7, 11, 13, 17, 19, 23, 29, 31}) {
        while (m % q == 0) {
            rad.push_back(q);
            m /= q;
        }
    }
    if (m != 1) return false;  // prime factor > 31
    // pair 3s with 5s (15), then 3s together (9), 5s alone
    while (e3 > 0 && e5 > 0) { rad.push_back(15); --e3; --e5; }
    while (e3 >= 2) { rad.push_back(9); e3 -= 2; }
    int left3 = e3, left5 = e5;
    // powers of two in 16s, remainder merged with a lone 3 or 5 when possible
    while (e2 >= 4) { rad.push_back(16); e2 -= 4; }
    if (left3) {
        if (e2 >= 2) { rad.push_back(12); e2 -= 2; }
        else if (e2 == 1) { rad.push_back(6); e2 -= 1; }
        else rad.push_back(3);
    }
    while (left5 > 0) {
        if (e2 >= 1) { rad.push_back(10); e2 -= 1; }
        else rad.push_back(5);
        --left5;
    }
    if (e2 == 3) rad.push_back(8);
    else if (e2 == 2) rad.push_back(4);
    else if (e2 == 1) rad.push_back(2);
    if (static_cast<int>(rad.size()) > kMaxStages) return false;
    p->nstages = static_cast<int>(rad.size());
    for (size_t i = 0; i < rad.size(); ++i) p->radix[i] = rad[i];
    return true;
}


// ---------------------------------------------------------------- codelets

template <int R, int DIR, class T>
__host__ __device__ __forceinline__ cx<T> root(int m) {
    // exp(DIR * 2 pi i m / R)
    return mk<T>(static_cast<T>(Root<R>::c(m)), static_cast<T>(DIR * Root<R>::s(m)));
}

template <int R, int DIR, class T>
__host__ __device__ __forceinline__ cx<T> twiddle_const(cx<T> v, int m) {
    // v * exp(DIR * 2 pi i m / R) with the trivial cases folded
    m %= R;
    if (m == 0) return v;
    if (4 * m == R) return mul_i<DIR>(v);
    if (2 * m == R) return mk<T>(-v.x, -v.y);
    if (4 * m == 3 * R) return mul_i<-DIR>(v);
    return v * root<R, DIR, T>(m);
}

template <int R, int DIR, class T>
struct Dft;

template <int DIR, class T>
struct Dft<1, DIR, T> {
    static __host__ __device__ __forceinline__ void run(cx<T>*) {}
};

template <int DIR, class T>
struct Dft<2, DIR, T> {
    static __host__ __device__ __forceinline__ void run(cx<T>* v) {
        const cx<T> a = v[0], b = v[1];
        v[0] = a + b;
        v[1] = a - b;
    }
};

template <int DIR, class T>
struct Dft<3, DIR, T> {
    static __host__ __device__ __forceinline__ void run(cx<T>* v) {
        const T h = static_cast<T>(0.8660254037844386467637232);
        const cx<T> t1 = v[1] + v[2];
        const cx<T> t2 = v[1] - v[2];
        const cx<T> m = mk<T>(v[0].x - static_cast<T>(0.5) * t1.x, v[0].y - static_cast<T>(0.5) * t1.y);
        const cx<T> nn = scale(mul_i<DIR>(t2), h);
        v[0] = v[0] + t1;
        v[1] = m + nn;
        v[2] = m - nn;
    }
};

template <int DIR, class T>
struct Dft<4, DIR, T> {
    static __host__ __device__ __forceinline__ void run(cx<T>* v) {
        const cx<T> t0 = v[0] + v[2], t1 = v[0] - v[2];
        const cx<T> t2 = v[1] + v[3], t3 = mul_i<DIR>(v[1] - v[3]);
        v[0] = t0 + t2;
        v[1] = t1 + t3;
        v[2] = t0 - t2;
        v[3] = t1 - t3;
    }
};

template <int DIR, class T>
struct Dft<5, DIR, T> {
    static __host__ __device__ __forceinline__ void run(cx<T>* v) {
        const T c1 = static_cast<T>(0.3090169943749474241022934);
        const T c2 = static_cast<T>(-0.8090169943749474241022934);
        const T s1 = static_cast<T>(0.9510565162951535721164393);
        const T s2 = static_cast<T>(0.5877852522924731291687060);
        const cx<T> t1 = v[1] + v[4], t2 = v[2] + v[3];
        const cx<T> t3 = v[1] - v[4], t4 = v[2] - v[3];
        const cx<T> b1 = v[0] + scale(t1, c1) + scale(t2, c2);
        const cx<T> b2 = v[0] + scale(t1, c2) + scale(t2, c1);
        const cx<T> d1 = mul_i<DIR>(scale(t3, s1) + scale(t4, s2));
        const cx<T> d2 = mul_i<DIR>(scale(t3, s2) - scale(t4, s1));
        v[0] = v[0] + t1 + t2;
        v[1] = b1 + d1;
        v[4] = b1 - d1;
        v[2] = b2 + d2;
        v[3] = b2 - d2;
    }
};

// R = A * B by Cooley-Tukey inside registers: n = B a + b, k = k1 + A k2.
template <int A, int B, int DIR, class T>
struct DftCT {
    static __host__ __device__ __forceinline__ void run(cx<T>* v) {
        constexpr int R = A * B;
        cx<T> y[R];  // y[b * A + k1]
#pragma unroll
        for (int b = 0; b < B; ++b) {
            cx<T> u[A];
#pragma unroll
            for (int a = 0; a < A; ++a) u[a] = v[B * a + b];
            Dft<A, DIR, T>::run(u);
#pragma unroll
            for (int k1 = 0; k1 < A; ++k1) y[b * A + k1] = twiddle_const<R, DIR>(u[k1], b * k1);
        }
#pragma unroll
        for (int k1 = 0; k1 < A; ++k1) {
            cx<T> u[B];
#pragma unroll
            for (int b = 0; b < B; ++b) u[b] = y[b * A + k1];
            Dft<B, DIR, T>::run(u);
#pragma unroll
            for (int k2 = 0; k2 < B; ++k2) v[k1 + A * k2] = u[k2];
        }
    }
};

// R = A * B with gcd(A, B) = 1 by Good-Thomas (prime-factor) indexing: no internal
// twiddles.  n = (B a + A b) mod R, k = (B <B^-1>_A k1 + A <A^-1>_B k2) mod R, so
// exp(2 pi i n k / R) = exp(2 pi i a k1 / A) exp(2 pi i b k2 / B).
template <int A, int B, int DIR, class T>
struct DftPFA {
    static constexpr int inv_mod(int x, int m) {
        int r = 1;
        while ((x * r) % m != 1) ++r;
        return r;
    }
    static __host__ __device__ __forceinline__ void run(cx<T>* v) {
        constexpr int R = A * B;
        constexpr int CA = B * inv_mod(B % A, A), CB = A * inv_mod(A % B, B);
        cx<T> y[R];  // y[k1 * B + b]
#pragma unroll
        for (int b = 0; b < B; ++b) {
            cx<T> u[A];
#pragma unroll
            for (int a = 0; a < A; ++a) u[a] = v[(B * a + A * b) % R];
            Dft<A, DIR, T>::run(u);
#pragma unroll
            for (int k1 = 0; k1 < A; ++k1) y[k1 * B + b] = u[k1];
        }
#pragma unroll
        for (int k1 = 0; k1 < A; ++k1) {
            Dft<B, DIR, T>::run(y + k1 * B);
#pragma unroll
            for (int k2 = 0; k2 < B; ++k2) v[(CA * k1 + CB * k2) % R] = y[k1 * B + k2];
        }
    }
};

// direct DFT for the odd primes 7..31
template <int R, int DIR, class T>
struct DftDirect {
    static __host__ __device__ __forceinline__ void run(cx<T>* v) {
        cx<T> out[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            cx<T> acc = v[0];
#pragma unroll
            for (int t = 1; t < R; ++t) acc = acc + twiddle_const<R, DIR>(v[t], t * k);
            out[k] = acc;
        }
#pragma unroll
        for (int k = 0; k < R; ++k) v[k] = out[k];
    }
};

template <int DIR, class T> struct Dft<6, DIR, T> : DftPFA<2, 3, DIR, T> {};
template <int DIR, class T> struct Dft<8, DIR, T> : DftCT<2, 4, DIR, T> {};
template <int DIR, class T> struct Dft<9, DIR, T> : DftCT<3, 3, DIR, T> {};
template <int DIR, class T> struct Dft<10, DIR, T> : DftPFA<2, 5, DIR, T> {};
template <int DIR, class T> struct Dft<12, DIR, T> : DftPFA<3, 4, DIR, T> {};
template <int DIR, class T> struct Dft<14, DIR, T> : DftPFA<2, 7, DIR, T> {};
template <int DIR, class T> struct Dft<15, DIR, T> : DftPFA<3, 5, DIR, T> {};
template <int DIR, class T> struct Dft<16, DIR, T> : DftCT<4, 4, DIR, T> {};
template <int DIR, class T> struct Dft<7, DIR, T> : DftDirect<7, DIR, T> {};
template <int DIR, class T> struct Dft<11, DIR, T> : DftDirect<11, DIR, T> {};
template <int DIR, class T> struct Dft<13, DIR, T> : DftDirect<13, DIR, T> {};
template <int DIR, class T> struct Dft<17, DIR, T> : DftDirect<17, DIR, T> {};
template <int DIR, class T> struct Dft<19, DIR, T> : DftDirect<19, DIR, T> {};
template <int DIR, class T> struct Dft<23, DIR, T> : DftDirect<23, DIR, T> {};
template <int DIR, class T> struct Dft<29, DIR, T> : DftDirect<29, DIR, T> {};
template <int DIR, class T> struct Dft<31, DIR, T> : DftDirect<31, DIR, T> {};

// ------------------------------------------------------------------ stage

// One Stockham butterfly j of a stage with radix R, ns = product of earlier radices.
// ld(i) reads element i of the stage input, st(i, v) writes element i of the output.
template <int R, int DIR, class T, class Ld, class St>
__host__ __device__ __forceinline__ void butterfly(int j, int n, int ns, const cx<T>* __restrict__ tw, Ld ld, St st) {
    const int m = n / R;
    const int k = j % ns;
    cx<T> v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = ld(j + r * m);
    if (ns > 1) {
        const int step = (n / (ns * R)) * k;
#pragma unroll
        for (int r = 1; r < R; ++r) {
            cx<T> w = tw[r * step];
            if (DIR > 0) w.y = -w.y;
            v[r] = v[r] * w;
        }
    }
    Dft<R, DIR, T>::run(v);
    const int base = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) st(base + r * ns, v[r]);
}

template <int DIR, class T, class Ld, class St>
__host__ __device__ __forceinline__ void butterfly_any(int R, int j, int n, int ns, const cx<T>* __restrict__ tw, Ld ld,
                                              St st) {
    switch (R) {
        case 2: butterfly<2, DIR, T>(j, n, ns, tw, ld, st); break;
        case 3: butterfly<3, DIR, T>(j, n, ns, tw, ld, st); break;
        case 4: butterfly<4, DIR, T>(j, n, ns, tw, ld, st); break;
        case 5: butterfly<5, DIR, T>(j, n, ns, tw, ld, st); break;
        case 6: butterfly<6, DIR, T>(j, n, ns, tw, ld, st); break;
        case 7: butterfly<7, DIR, T>(j, n, ns, tw, ld, st); break;
        case 8: butterfly<8, DIR, T>(j, n, ns, tw, ld, st); break;
        case 9: butterfly<9, DIR, T>(j, n, ns, tw, ld, st); break;
        case 10: butterfly<10, DIR, T>(j, n, ns, tw, ld, st); break;
        case 11: butterfly<11, DIR, T>(j, n, ns, tw, ld, st); break;
        case 12: butterfly<12, DIR, T>(j, n, ns, tw, ld, st); break;
        case 13: butterfly<13, DIR, T>(j, n, ns, tw, ld, st); break;
        case 14: butterfly<14, DIR, T>(j, n, ns, tw, ld, st); break;
        case 15: butterfly<15, DIR, T>(j, n, ns, tw, ld, st); break;
        case 16: butterfly<16, DIR, T>(j, n, ns, tw, ld, st); break;
        case 17: butterfly<17, DIR, T>(j, n, ns, tw, ld, st); break;
        case 19: butterfly<19, DIR, T>(j, n, ns, tw, ld, st); break;
        case 23: butterfly<23, DIR, T>(j, n, ns, tw, ld, st); break;
        case 29: butterfly<29, DIR, T>(j, n, ns, tw, ld, st); break;
        case 31: butterfly<31, DIR, T>(j, n, ns, tw, ld, st); break;
        default: break;
    }
}

// Layouts of a batch of NB transforms of length n in shared memory.
// Column layout: element i of transform b at [i * NB + b] (b fastest; used for strips of columns).
// Row layout: element i of transform b at [b * n + i] (i fastest; used for contiguous rows).
struct ColLayout {
    int n, nb;
    __device__ __forceinline__ int at(int b, int i) const { return i * nb + b; }
};
struct RowLayout {
    int n, nb;
    __device__ __forceinline__ int at(int b, int i) const { return b * n + i; }
};

// Run all Stockham stages over a batch in shared memory, ping-ponging between
// buf0 and buf1 (both n * nb elements).  Returns the buffer holding the result.
// Thread mapping: for the column layout consecutive threads take consecutive
// transforms (b), for the row layout consecutive butterflies (j).
template <int DIR, class T, class Layout>
__device__ cx<T>* fft_batch(cx<T>* buf0, cx<T>* buf1, const Layout lay, const FftPlan& plan,
                            const cx<T>* __restrict__ tw) {
    const int n = lay.n, nb = lay.nb;
    cx<T>* src = buf0;
    cx<T>* dst = buf1;
    int ns = 1;
    for (int s = 0; s < plan.nstages; ++s) {
        const int R = plan.radix[s];
        const int per = n / R;
        const int total = per * nb;
        for (int t = threadIdx.x; t < total; t += blockDim.x) {
            int b, j;
            if constexpr (std::is_same<Layout, ColLayout>::value) {
                b = t % nb;
                j = t / nb;
            } else {
                b = t / per;
                j = t % per;
            }
            const cx<T>* s_ = src;
            cx<T>* d_ = dst;
            butterfly_any<DIR, T>(
                R, j, n, ns, tw, [&](int i) { return s_[lay.at(b, i)]; },
                [&](int i, cx<T> v) { d_[lay.at(b, i)] = v; });
        }
        __syncthreads();
        cx<T>* t = src;
        src = dst;
        dst = t;
        ns *= R;
    }
    return src;
}

}  // namespace holo_cuda
