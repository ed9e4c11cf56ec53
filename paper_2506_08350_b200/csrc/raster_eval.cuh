// Per-entry evaluation shared by the compositing kernel (composite.cu) and its
// backward (backward.cu): both must take the same accept decisions, so they
// stage identical records and run the identical instruction sequence.
//
// evaluate() of rasterizer.cpp:124-135 in fp32: d = pixel centre - mu (the centre
// offset formed in f64 per entry, tile-relative), form in the log2 domain with
// alpha folded into the exponent, a = min(2^(q + log2 alpha), alpha_clamp).
#pragma once

#include "kernels.cuh"

namespace holo_cuda {

// 2^x on the MUFU pipe (max rel. error 2^-22.5); x <= 0 here, results below 2^-126 flush to 0.
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// One staged entry: 48 bytes, read with three 16-byte shared loads from one base;
// its accept box lives in a separate array read only by the ballot test.
struct alignas(16) Staged {
    float4 a;  // mx, my, ca, cb   (centre relative to the tile origin; conic, log2-scaled)
    float4 b;  // cc, log2(alpha), col0 re, col0 im
    float4 c;  // col1 re, col1 im, col2 re, col2 im
};

// Record of Gaussian r for the tile at (px0, py0); alpha already carries rho in
// soft mode.  box = (xlo, xhi, ylo, yhi) of the accept ellipse, tile-relative.
__device__ __forceinline__ void stage_entry(const GRec& r, int px0, int py0, float alpha, Staged& st, float4& box) {
    const float mx = static_cast<float>(r.mu_x - static_cast<double>(px0));
    const float my = static_cast<float>(r.mu_y - static_cast<double>(py0));
    st.a = make_float4(mx, my, r.ca, r.cb);
    st.b = make_float4(r.cc, log2f(alpha), r.col[0], r.col[1]);
    st.c = make_float4(r.col[2], r.col[3], r.col[4], r.col[5]);
    box = make_float4(mx - r.hx, mx + r.hx, my - r.hy, my + r.hy);
}

// alpha of entry e at pixel centre (fx, fy), tile-relative; B receives e->b.
__device__ __forceinline__ float eval_alpha(const Staged* e, float fx, float fy, float clamp, float4& B) {
    const float4 A = e->a;
    B = e->b;
    const cx<float> d = mk(fx, fy) - mk(A.x, A.y);  // one FADD2
    const float dx = d.x, dy = d.y;
    const float t = fmaf(A.w, dy, A.z * dx);
    const float u = fmaf(dx, t, B.y);
    const float q = fmaf(B.x * dy, dy, u);
    return fminf(ex2_approx(q), clamp);
}

// acc_c += w * (amp_c cos phi_c, amp_c sin phi_c): one FFMA2 per channel
__device__ __forceinline__ cx<float> axpy(float w, float re, float im, cx<float> acc) {
    return f32x2::unpack(f32x2::fma(f32x2::pack(w, w), f32x2::pack(re, im), f32x2::pack(acc.x, acc.y)));
}

// acc[c] += w * amp_c e^{i phi_c}
template <int C>
__device__ __forceinline__ void blend(const Staged* e, const float4& B, float w, cx<float> (&acc)[C]) {
    acc[0] = axpy(w, B.z, B.w, acc[0]);
    if constexpr (C > 1) {
        const float4 Cc = e->c;
        acc[1 % C] = axpy(w, Cc.x, Cc.y, acc[1 % C]);
        if constexpr (C > 2) acc[2 % C] = axpy(w, Cc.z, Cc.w, acc[2 % C]);
    }
}

// blend with the channel-1/2 phasors already loaded (Cc = the record's c)
template <int C>
__device__ __forceinline__ void blend_c(const float4& B, const float4& Cc, float w, cx<float> (&acc)[C]) {
    acc[0] = axpy(w, B.z, B.w, acc[0]);
    if constexpr (C > 1) {
        acc[1 % C] = axpy(w, Cc.x, Cc.y, acc[1 % C]);
        if constexpr (C > 2) acc[2 % C] = axpy(w, Cc.z, Cc.w, acc[2 % C]);
    }
}

// 16-byte shared load from a shared-window address
__device__ __forceinline__ float4 lds128(unsigned addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// does the accept box meet the warp's block of pixel centres [bxlo, bxhi] x [bylo, byhi]?
__device__ __forceinline__ bool box_hits(const float4& bb, float bxlo, float bxhi, float bylo, float byhi) {
    return !(bb.y < bxlo || bb.x > bxhi || bb.w < bylo || bb.z > byhi);
}

// w if (a > thr) and (T >= eps), else 0: the accept decision of eval_alpha's
// callers as one compare with the other folded in and one select
__device__ __forceinline__ float accept_weight(float a, float thr, float T, float eps, float w) {
    float r;
    asm("{\n.reg .pred l, p;\nsetp.ge.f32 l, %2, %4;\nsetp.gt.and.f32 p, %1, %3, l;\nselp.f32 %0, %5, 0f00000000, p;\n}"
        : "=f"(r)
        : "f"(a), "f"(T), "f"(thr), "f"(eps), "f"(w));
    return r;
}

}  // namespace holo_cuda
