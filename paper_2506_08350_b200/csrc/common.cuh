// Shared device/host helpers for libholo_cuda (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "holo_cuda.h"

namespace holo_cuda {

// Error carried across the C-ABI as (status code, message).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define HC_CUDA(expr)                                                                                      \
    do {                                                                                                   \
        cudaError_t hc_e_ = (expr);                                                                        \
        if (hc_e_ != cudaSuccess)                                                                          \
            throw ::holo_cuda::Error(hc_e_ == cudaErrorMemoryAllocation ? HOLO_ERR_OOM : HOLO_ERR_CUDA,  \
                                     std::string(#expr) + ": " + cudaGetErrorString(hc_e_));               \
    } while (0)

#define HC_LAUNCHED(ctx)                                  \
    do {                                                  \
        HC_CUDA(cudaGetLastError());                      \
        (ctx)->note_launch();                             \
    } while (0)

inline void config_error(const std::string& msg) { throw Error(HOLO_ERR_CONFIG, msg); }

// Complex number in interleaved (re, im) layout, 8- or 16-byte aligned like float2/double2.
template <class T>
struct alignas(2 * sizeof(T)) cx {
    T x, y;
};

template <class T>
__host__ __device__ __forceinline__ cx<T> mk(T a, T b) {
    cx<T> r;
    r.x = a;
    r.y = b;
    return r;
}
template <class T>
__host__ __device__ __forceinline__ cx<T> operator+(cx<T> a, cx<T> b) {
    return mk(a.x + b.x, a.y + b.y);
}
template <class T>
__host__ __device__ __forceinline__ cx<T> operator-(cx<T> a, cx<T> b) {
    return mk(a.x - b.x, a.y - b.y);
}
template <class T>
__host__ __device__ __forceinline__ cx<T> operator*(cx<T> a, cx<T> b) {
    return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <class T>
__host__ __device__ __forceinline__ cx<T> scale(cx<T> a, T s) {
    return mk(a.x * s, a.y * s);
}
template <class T>
__host__ __device__ __forceinline__ cx<T> conj(cx<T> a) {
    return mk(a.x, -a.y);
}
// a * (dir * i): dir = +1 multiplies by i, -1 by -i
template <int DIR, class T>
__host__ __device__ __forceinline__ cx<T> mul_i(cx<T> a) {
    return DIR > 0 ? mk(-a.y, a.x) : mk(a.y, -a.x);
}
// c + a * b
template <class T>
__host__ __device__ __forceinline__ cx<T> cfma(cx<T> a, cx<T> b, cx<T> c) {
    return c + a * b;
}

// ---- fp32 complex arithmetic on the packed fp32x2 pipe (sm_100: FADD2 / FMUL2 /
// FFMA2, one instruction for both lanes).  ptxas folds the lane swaps, partial
// negations and scalar broadcasts below into operand modifiers, so
//   a +- b        1 instruction (2 scalar)
//   a * s, s real 1           (2)
//   a * b         2: a.x-broadcast product, then (-a.y, a.x) fused with b.y   (4)
//   c + a * b     2                                                           (4 + 2)
// Lane results are the IEEE round-to-nearest ones of the scalar operations.
namespace f32x2 {
__device__ __forceinline__ unsigned long long pack(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ cx<float> unpack(unsigned long long r) {
    cx<float> v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ unsigned long long add(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long sub(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long mul(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long fma(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
}  // namespace f32x2

__host__ __device__ __forceinline__ cx<float> operator+(cx<float> a, cx<float> b) {
#ifdef __CUDA_ARCH__
    return f32x2::unpack(f32x2::add(f32x2::pack(a.x, a.y), f32x2::pack(b.x, b.y)));
#else
    return mk(a.x + b.x, a.y + b.y);
#endif
}
__host__ __device__ __forceinline__ cx<float> operator-(cx<float> a, cx<float> b) {
#ifdef __CUDA_ARCH__
    return f32x2::unpack(f32x2::sub(f32x2::pack(a.x, a.y), f32x2::pack(b.x, b.y)));
#else
    return mk(a.x - b.x, a.y - b.y);
#endif
}
__host__ __device__ __forceinline__ cx<float> operator*(cx<float> a, cx<float> b) {
#ifdef __CUDA_ARCH__
    const unsigned long long t = f32x2::mul(f32x2::pack(a.x, a.y), f32x2::pack(b.x, b.x));
    return f32x2::unpack(f32x2::fma(f32x2::pack(-a.y, a.x), f32x2::pack(b.y, b.y), t));
#else
    return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
#endif
}
__host__ __device__ __forceinline__ cx<float> scale(cx<float> a, float s) {
#ifdef __CUDA_ARCH__
    return f32x2::unpack(f32x2::mul(f32x2::pack(a.x, a.y), f32x2::pack(s, s)));
#else
    return mk(a.x * s, a.y * s);
#endif
}
__host__ __device__ __forceinline__ cx<float> cfma(cx<float> a, cx<float> b, cx<float> c) {
#ifdef __CUDA_ARCH__
    const unsigned long long t = f32x2::fma(f32x2::pack(a.x, a.y), f32x2::pack(b.x, b.x), f32x2::pack(c.x, c.y));
    return f32x2::unpack(f32x2::fma(f32x2::pack(-a.y, a.x), f32x2::pack(b.y, b.y), t));
#else
    return c + a * b;
#endif
}

template <class T>
__host__ __device__ __forceinline__ T cdiv(T a, T b) {
    return (a + b - 1) / b;
}

}  // namespace holo_cuda
