// K1 preprocess: per-Gaussian projection in f64 (sm_100a).
//
// Restates detail::project_gaussian (proj/src/rasterizer.cpp:10-70) with
// covariance_3d / quat_to_rot (scene.cpp:74-82,125-130), the sigmoid of
// common.hpp:32-40, ste_assign's argmax (scene.cpp:132-152) and tile_span
// (rasterizer.cpp:106-113).  This translation unit is compiled with
// --fmad=false and follows the reference's expression order (3x3 products as
// left-to-right inner sums, oracle/shim/Eigen/Dense) so that the depth keys,
// footprints and tile spans -- and therefore the per-tile work lists -- match
// the reference bit for bit.  One thread per Gaussian; f64 scene in, a 64-byte
// fp32 compositing record plus binning metadata out.
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "bulk.cuh"
#include "kernels.cuh"

namespace holo_cuda {

// rot_cam_to_world = Rz Ry Rx (camera.cpp:5-14) on the host with libm trig, transposed.
void host_world_to_cam(const holo_camera& cam, double wc[9]) {
    const double cx = std::cos(cam.pose[3]), sx = std::sin(cam.pose[3]);
    const double cy = std::cos(cam.pose[4]), sy = std::sin(cam.pose[4]);
    const double cz = std::cos(cam.pose[5]), sz = std::sin(cam.pose[5]);
    const double rx[9] = {1, 0, 0, 0, cx, -sx, 0, sx, cx};
    const double ry[9] = {cy, 0, sy, 0, 1, 0, -sy, 0, cy};
    const double rz[9] = {cz, -sz, 0, sz, cz, 0, 0, 0, 1};
    auto mul = [](const double* a, const double* b, double* c) {
        double t[9];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                t[i * 3 + j] = (a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j]) + a[i * 3 + 2] * b[2 * 3 + j];
        for (int i = 0; i < 9; ++i) c[i] = t[i];
    };
    double t[9], r[9];
    mul(rz, ry, t);
    mul(t, rx, r);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) wc[i * 3 + j] = r[j * 3 + i];
}

namespace {

struct PreArgs {
    const double* positions;
    const double* rotations;
    const double* log_scales;
    const double* amplitudes;
    const double* opacity;
    const double* phases;
    const double* plane_logits;
    size_t n;
    int L;
    CameraConsts cam;
    double near_clip, dilation, alpha_floor, radius_form_cap, plane_eps, soft_tau;
    double inv_tile;  // 1 / tile when the tile is a power of two (exact), else 0
    int soft, tile, tiles_x, tiles_y;
    int staged;  // full slices are staged in shared memory with bulk copies
};

__device__ __forceinline__ double sigmoid_ref(double x) {
    if (x >= 0.0) {
        const double e = exp(-x);
        return 1.0 / (1.0 + e);
    }
    const double e = exp(x);
    return e / (1.0 + e);
}

// PROJ: also fill the full f64 detail::Projected record (HOLO_OUT_PROJECTED); the
// render path compiles it out, which keeps the kernel at 64 registers.
#ifndef HOLO_PRE_NT
#define HOLO_PRE_NT 64  // 12 CTAs of 64 per SM: C3 0.091 -> 0.089 ms, C5 0.465 -> 0.442 ms against 6 of 128
#endif
#ifndef HOLO_PRE_MINB
#define HOLO_PRE_MINB (768 / HOLO_PRE_NT)  // 80 registers: no spills (measured best)
#endif
constexpr int kPreNT = HOLO_PRE_NT;
// Staged scene slice of one CTA, in doubles per Gaussian: positions 3, rotations 4,
// log-scales 3, amplitudes 3, opacity 1, phases 3, then the L plane logits.
constexpr int kStageFixed = 17;
inline size_t stage_bytes(int L) { return sizeof(double) * kPreNT * (kStageFixed + static_cast<size_t>(L)); }

// One CTA's view of the scene arrays for its current slice of kPreNT Gaussians:
// shared-memory copies (staged slices) or the global arrays.
struct Slice {
    const double *pos, *rot, *ls, *amp, *op, *ph, *lg;
};

// Issue the bulk copies of slice `sl` into buffer `buf` (one thread).
__device__ __forceinline__ void stage_slice(const PreArgs& a, size_t sl, double* buf, unsigned long long* bar,
                                            bool logits) {
    constexpr unsigned kNT = kPreNT;
    const size_t i0 = sl * kNT;
    const unsigned lg_bytes = logits ? 8u * kNT * static_cast<unsigned>(a.L) : 0u;
    bulk::mbar_expect_tx(bar, 8u * kNT * kStageFixed + lg_bytes);
    bulk::bulk_g2s(buf, a.positions + 3 * i0, 24 * kNT, bar);
    bulk::bulk_g2s(buf + 3 * kNT, a.rotations + 4 * i0, 32 * kNT, bar);
    bulk::bulk_g2s(buf + 7 * kNT, a.log_scales + 3 * i0, 24 * kNT, bar);
    bulk::bulk_g2s(buf + 10 * kNT, a.amplitudes + 3 * i0, 24 * kNT, bar);
    bulk::bulk_g2s(buf + 13 * kNT, a.opacity + i0, 8 * kNT, bar);
    bulk::bulk_g2s(buf + 14 * kNT, a.phases + 3 * i0, 24 * kNT, bar);
    if (logits) bulk::bulk_g2s(buf + 17 * kNT, a.plane_logits + i0 * a.L, lg_bytes, bar);
}

template <bool PROJ>
__device__ __forceinline__ void project_one(const PreArgs& a, const PreOut& o, size_t i, int t, const Slice& v) {
    const int L = a.L;
    const double *rot_b = v.rot, *amp_b = v.amp, *lg_b = v.lg, *pos_b = v.pos, *ls_b = v.ls, *op_b = v.op,
                 *ph_b = v.ph;

    // ---- scene validation (scene.cpp:19-32), over every Gaussian
    const double* q = rot_b + 4 * t;
    const double q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
    const double qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    unsigned bad = 0;
    if (!(qn > 1e-8)) bad |= 1u;
    const double* amp = amp_b + 3 * t;
    if (amp[0] < 0.0 || amp[1] < 0.0 || amp[2] < 0.0) bad |= 2u;
    if (bad) atomicOr(o.flags, bad);

    // ---- plane assignment (compute_rho, rasterizer.cpp:81-99; ste_assign scene.cpp:132-152)
    const double* lg = lg_b + static_cast<size_t>(t) * L;
    // The reference's strict-'>' scan from plane 0 yields the first index of the
    // largest non-NaN logit, or 0 when logit 0 is NaN (NaNs never win).  The same
    // result is formed here reading the planes in an order rotated by the thread
    // index, so that a warp's reads of its 32 staged rows (L doubles apart) fall in
    // distinct shared-memory banks instead of L-way conflicting ones.
    int best = 0;
    {
        int bl = -1;
        double bv = 0.0;
        int l = L > 0 ? t % L : 0;
        for (int k = 0; k < L; ++k) {
            const double v = lg[l];
            if (!isnan(v) && (bl < 0 || v > bv || (v == bv && l < bl))) {
                bv = v;
                bl = l;
            }
            if (++l == L) l = 0;
        }
        best = (bl < 0 || isnan(lg[0])) ? 0 : bl;
    }
    o.plane[i] = best;
    unsigned long long mask = 0;
    int nplanes = 0;
    if (a.soft) {
        const double top = lg[best];
        double denom = 0.0;
        for (int l = 0; l < L; ++l) denom += exp((lg[l] - top) / a.soft_tau);
        for (int l = 0; l < L; ++l) {
            const double r = exp((lg[l] - top) / a.soft_tau) / denom;
            if (o.rho) o.rho[i * L + l] = r;
            if (r > 0.0 && l < 64) {  // soft gate is 0 (rasterizer.cpp:175)
                mask |= 1ull << l;
                ++nplanes;
            }
        }
    } else {
        if (o.rho)
            for (int l = 0; l < L; ++l) o.rho[i * L + l] = (l == best) ? 1.0 : 0.0;
        nplanes = (1.0 > a.plane_eps) ? 1 : 0;  // one-hot weight vs the gate (:176-186)
        mask = (best < 64) ? (1ull << best) : 0ull;
    }
    if (o.pmask) o.pmask[i] = mask;
    if constexpr (!PROJ) {
        // plane-sharded frame (hard assignment): a Gaussian of another rank's
        // planes emits no entry here, so its projection is skipped
        if (o.slots && (best < o.pb || best >= o.pe)) {
            o.count[i] = 0;
            o.rect[i] = make_int4(0, 0, 0, 0);
            if (o.touched) o.touched[i] = 0;
            return;
        }
    }

    // ---- projection (rasterizer.cpp:10-70)
    holo_projected p;
    p.valid = 0;
    p.n = static_cast<int>(i);
    p.mu_x = p.mu_y = p.inv00 = p.inv01 = p.inv11 = p.radius = 0.0;
    p.xc = p.yc = p.zc = p.alpha_sig = 0.0;
    for (int c = 0; c < 3; ++c) p.amp[c] = p.phase[c] = 0.0;
    p.plane = best;
    p.pad_ = 0;

    const double* xw = pos_b + 3 * t;
    const double d0 = xw[0] - a.cam.pos[0], d1 = xw[1] - a.cam.pos[1], d2 = xw[2] - a.cam.pos[2];
    const double* W = a.cam.wc;
    const double xc0 = (W[0] * d0 + W[1] * d1) + W[2] * d2;
    const double xc1 = (W[3] * d0 + W[4] * d1) + W[5] * d2;
    const double xc2 = (W[6] * d0 + W[7] * d1) + W[8] * d2;

    int4 rect = make_int4(0, 0, 0, 0);
    unsigned count = 0;
    bool valid = false;
    double alpha = 0.0, radius = 0.0;
    double inv00 = 0.0, inv01 = 0.0, inv11 = 0.0;
    double cov00_out = 0.0, cov11_out = 0.0, log_ratio2 = 0.0;
    if (xc2 > a.near_clip) {
        p.xc = xc0;
        p.yc = xc1;
        p.zc = xc2;
        const double f = a.cam.focal;
        const double iz = 1.0 / xc2;
        p.mu_x = f * xc0 * iz + a.cam.ppx;
        p.mu_y = f * xc1 * iz + a.cam.ppy;
        double J[6] = {0, 0, 0, 0, 0, 0};
        J[0] = f * iz;
        J[4] = f * iz;
        J[2] = -f * xc0 * iz * iz;
        J[5] = -f * xc1 * iz * iz;

        // covariance_3d: R from the normalised quaternion, M = R diag(exp(s)), Sigma = M M^T
        const double w = q0 / qn, x = q1 / qn, y = q2 / qn, z = q3 / qn;
        const double R[9] = {
            1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z),       2.0 * (x * z + w * y),
            2.0 * (x * y + w * z),       1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
            2.0 * (x * z - w * y),       2.0 * (y * z + w * x),       1.0 - 2.0 * (x * x + y * y),
        };
        const double* ls = ls_b + 3 * t;
        double Mq[9];
        for (int k = 0; k < 3; ++k) {
            const double e = exp(ls[k]);
            for (int r = 0; r < 3; ++r) Mq[r * 3 + k] = R[r * 3 + k] * e;
        }
        double S[9];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                S[r * 3 + c] = (Mq[r * 3 + 0] * Mq[c * 3 + 0] + Mq[r * 3 + 1] * Mq[c * 3 + 1]) + Mq[r * 3 + 2] * Mq[c * 3 + 2];
        // M = J W (2x3), T = M Sigma, cov = T M^T
        double M[6], T[6];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c)
                M[r * 3 + c] = (J[r * 3 + 0] * W[0 * 3 + c] + J[r * 3 + 1] * W[1 * 3 + c]) + J[r * 3 + 2] * W[2 * 3 + c];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c)
                T[r * 3 + c] = (M[r * 3 + 0] * S[0 * 3 + c] + M[r * 3 + 1] * S[1 * 3 + c]) + M[r * 3 + 2] * S[2 * 3 + c];
        double cov00 = (T[0] * M[0] + T[1] * M[1]) + T[2] * M[2];
        const double cov01 = (T[0] * M[3] + T[1] * M[4]) + T[2] * M[5];
        double cov11 = (T[3] * M[3] + T[4] * M[4]) + T[5] * M[5];
        cov00 += a.dilation;
        cov11 += a.dilation;
        cov00_out = cov00;
        cov11_out = cov11;
        const double det = cov00 * cov11 - cov01 * cov01;
        if (det > 0.0 && isfinite(det)) {
            const double idet = 1.0 / det;
            inv00 = cov11 * idet;
            inv01 = -cov01 * idet;
            inv11 = cov00 * idet;
            p.inv00 = inv00;
            p.inv01 = inv01;
            p.inv11 = inv11;
            alpha = sigmoid_ref(op_b[t]);
            p.alpha_sig = alpha;
            if (!(a.alpha_floor > 0.0) || alpha > a.alpha_floor) {
                // 2 ln(alpha / floor): the radius cap's c2 and the accept box's F
                if (a.alpha_floor > 0.0) log_ratio2 = 2.0 * log(alpha / a.alpha_floor);
                double form_cap = a.radius_form_cap;
                if (form_cap <= 0.0) {
                    form_cap = 9.0;
                    if (a.alpha_floor > 0.0) form_cap = form_cap < log_ratio2 ? log_ratio2 : form_cap;
                }
                const double mid = 0.5 * (cov00 + cov11);
                const double disc = mid * mid - det;
                const double lambda_max = mid + sqrt(disc > 0.0 ? disc : 0.0);
                radius = sqrt(form_cap * lambda_max);
                p.radius = radius;
                const double* ph = ph_b + 3 * t;
                for (int c = 0; c < 3; ++c) {
                    p.amp[c] = amp[c];
                    p.phase[c] = ph[c];
                }
                p.valid = 1;
                valid = true;
            }
        }
    }

    GRec r;
    r.mu_x = p.mu_x;
    r.mu_y = p.mu_y;
    const double k = -0.5 * 1.4426950408889634073599;  // -log2(e) / 2
    r.ca = static_cast<float>(k * inv00);
    r.cb = static_cast<float>(k * 2.0 * inv01);
    r.cc = static_cast<float>(k * inv11);
    r.alpha = static_cast<float>(alpha);
    // Accept region a = alpha g > floor is the ellipse d^T cov^-1 d < F, F = 2 ln(alpha/floor);
    // its bounding box has half-widths sqrt(F cov_xx), sqrt(F cov_yy).  Slightly
    // widened so fp32 evaluation at the boundary is never culled.
    r.hx = r.hy = INFINITY;
    if (valid && a.alpha_floor > 0.0) {
        const double F = log_ratio2;
        r.hx = static_cast<float>(sqrt(F * cov00_out) * 1.0001 + 1e-3);
        r.hy = static_cast<float>(sqrt(F * cov11_out) * 1.0001 + 1e-3);
    }
    for (int c = 0; c < 6; ++c) r.col[c] = 0.0f;
    if (valid) {
        for (int c = 0; c < 3; ++c) {
            double s, co;
            sincos(p.phase[c], &s, &co);
            r.col[2 * c] = static_cast<float>(p.amp[c] * co);
            r.col[2 * c + 1] = static_cast<float>(p.amp[c] * s);
        }
        // tile_span (rasterizer.cpp:106-113)
        // the tile is a power of two, so x / tile == x * (1 / tile) exactly, and
        // floor-then-convert is one rounding conversion (both saturate alike):
        // bit-identical spans with fewer XU-pipe instructions (the kernel's limiter)
        const double it = a.inv_tile;
        const auto span = [&](double v) { return __double2int_rd(it > 0.0 ? v * it : v / a.tile); };
        int x0 = span(p.mu_x - radius);
        int x1 = span(p.mu_x + radius) + 1;
        int y0 = span(p.mu_y - radius);
        int y1 = span(p.mu_y + radius) + 1;
        x0 = x0 > 0 ? x0 : 0;
        y0 = y0 > 0 ? y0 : 0;
        x1 = x1 < a.tiles_x ? x1 : a.tiles_x;
        y1 = y1 < a.tiles_y ? y1 : a.tiles_y;
        if (x0 < x1 && y0 < y1) {
            rect = make_int4(x0, x1, y0, y1);
            count = static_cast<unsigned>(nplanes) * static_cast<unsigned>((x1 - x0) * (y1 - y0));
        }
        atomicAdd(o.num_valid, 1u);
        // bucket counting for hard assignment (see PreOut): the slot atomics are
        // issued together and their latency hides behind the other warps' math
        if (o.slots && count > 0 && best >= o.pb && best < o.pe) {
            const int w = x1 - x0, n = static_cast<int>(count);
            const int b0 = (best - o.pb) * o.num_tiles + y0 * a.tiles_x + x0;
            // the k-th tile of the span, row-major: offsets stepped, no divisions
            const int row_skip = a.tiles_x - w;
            if (n <= kSlots) {
                unsigned s[kSlots];
                int off = 0, cx = 0;
#pragma unroll
                for (int k = 0; k < kSlots; ++k) {
                    if (k < n) s[k] = atomicAdd(o.bcount + b0 + off, 1u);
                    ++off;
                    if (++cx == w) {
                        cx = 0;
                        off += row_skip;
                    }
                }
#pragma unroll
                for (int k = 0; k < kSlots; ++k)
                    if (k < n) o.slots[static_cast<size_t>(k) * a.n + i] = s[k];
            } else {
                for (int y = y0; y < y1; ++y)
                    for (int x = 0; x < w; ++x) atomicAdd(o.bbig + b0 + (y - y0) * a.tiles_x + x, 1u);
            }
        }
    }
    o.rec[i] = r;
    o.rect[i] = rect;
    o.count[i] = count;
    o.zc[i] = p.zc;
    if (o.touched) o.touched[i] = count > 0 ? 1 : 0;
    if constexpr (PROJ) o.projected[i] = p;
}

// One CTA per slice of kPreNT Gaussians: a full slice of the seven f64 scene
// arrays lands in shared memory by bulk copies on one mbarrier -- one round trip
// of memory latency per CTA, contiguous transfers instead of 24-64 B strided
// per-thread reads, and no chain of dependent loads behind the projection's
// branches; the resident CTAs of an SM overlap one another's copies and math.
// (Measured against a persistent, double-buffered variant, which lost: 0.133 vs
// 0.092 ms at C3.)
template <bool PROJ>
__global__ void __launch_bounds__(kPreNT, PROJ ? 1 : HOLO_PRE_MINB) k_preprocess(PreArgs a, PreOut o) {
    extern __shared__ __align__(16) double s_scene[];
    __shared__ unsigned long long s_bar;
    constexpr unsigned kNT = kPreNT;
    const int t = threadIdx.x;
    const size_t sl = blockIdx.x, i0 = sl * kNT;
    Slice v;
    if (a.staged && i0 + kNT <= a.n) {
        if (t == 0) {
            bulk::mbar_init(&s_bar, 1);
            bulk::mbar_init_fence();
        }
        __syncthreads();
        if (t == 0) stage_slice(a, sl, s_scene, &s_bar, true);
        const double* s = s_scene;
        v = Slice{s, s + 3 * kNT, s + 7 * kNT, s + 10 * kNT, s + 13 * kNT, s + 14 * kNT, s + 17 * kNT};
        bulk::mbar_wait(&s_bar, 0);
    } else {
        v = Slice{a.positions + 3 * i0, a.rotations + 4 * i0, a.log_scales + 3 * i0, a.amplitudes + 3 * i0,
                  a.opacity + i0, a.phases + 3 * i0, a.plane_logits + i0 * a.L};
    }
    if (i0 + t < a.n) project_one<PROJ>(a, o, i0 + t, t, v);
}

}  // namespace

void preprocess(holo_ctx* ctx, const CameraConsts& cc, const holo_raster_settings& st, double near_clip, int L,
                int tiles_x, int tiles_y, const PreOut& out) {
    if (ctx->n == 0) return;
    PreArgs a;
    a.positions = ctx->d_positions;
    a.rotations = ctx->d_rotations;
    a.log_scales = ctx->d_log_scales;
    a.amplitudes = ctx->d_amplitudes;
    a.opacity = ctx->d_opacity;
    a.phases = ctx->d_phases;
    a.plane_logits = ctx->d_plane_logits;
    a.n = ctx->n;
    a.L = L;
    a.cam = cc;
    a.near_clip = near_clip;
    a.dilation = st.dilation;
    a.alpha_floor = st.alpha_floor;
    a.radius_form_cap = st.radius_form_cap;
    a.plane_eps = st.plane_eps;
    a.soft_tau = st.soft_tau;
    a.soft = st.soft_assignment;
    a.tile = st.tile;
    a.inv_tile = (st.tile > 0 && (st.tile & (st.tile - 1)) == 0) ? 1.0 / st.tile : 0.0;
    a.tiles_x = tiles_x;
    a.tiles_y = tiles_y;
    // staging needs 16-byte aligned slices (every array is its own allocation) and
    // a slice that leaves shared memory for several resident CTAs
    static const bool env_off = [] {
        const char* e = std::getenv("HOLO_PRE_STAGED");
        return e && e[0] == '0';
    }();
    const void* arrs[7] = {a.positions, a.rotations, a.log_scales, a.amplitudes, a.opacity, a.phases, a.plane_logits};
    bool aligned = true;
    for (const void* p : arrs) aligned = aligned && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
    const size_t smem = stage_bytes(L);
    a.staged = !env_off && aligned && smem <= 96 * 1024;
    const size_t dyn = a.staged ? smem : 0;
    const unsigned grid = static_cast<unsigned>((ctx->n + kPreNT - 1) / kPreNT);
    auto launch = [&](auto kernel) {
        if (dyn > 48 * 1024)
            HC_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn)));
        kernel<<<grid, kPreNT, dyn, ctx->stream>>>(a, out);
    };
    if (out.projected)
        launch(k_preprocess<true>);
    else
        launch(k_preprocess<false>);
    HC_LAUNCHED(ctx);
}

}  // namespace holo_cuda
