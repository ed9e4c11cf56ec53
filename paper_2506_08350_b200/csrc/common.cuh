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

template <class T>
__host__ __device__ __forceinline__ T cdiv(T a, T b) {
    return (a + b - 1) / b;
}

}  // namespace holo_cuda
