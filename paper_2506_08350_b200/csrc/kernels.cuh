// Internal kernel-side declarations shared by the libholo_cuda translation units.
#pragma once

#include <vector>

#include "context.h"

namespace holo_cuda {

// Transfer function H_z(fx, fy) (propagation.cpp:18-54) for one (plane, channel).
// The band test is done in f64 with the reference's expression order
// ((1/l^2 - fx^2) - fy^2 < 0 -> 0; __d*_rn keeps it uncontracted).  The f64
// variant evaluates the reference phase 2 pi z sqrt(arg) directly; the f32
// variant uses the cancellation-free split
//   2 pi z sqrt(1/l^2 - f^2) = 2 pi z / l  -  2 pi z f^2 / (1/l + sqrt(1/l^2 - f^2))
// with the first term reduced mod 2 pi on the host in f64 (phase0), so only a
// residual of at most a few hundred radians is formed in fp32.
template <class T>
__device__ __forceinline__ cx<T> tf_value(const TfChan& p, double fx, double fy);

template <>
__device__ __forceinline__ cx<double> tf_value<double>(const TfChan& p, double fx, double fy) {
    const double arg = __dsub_rn(__dsub_rn(p.inv_l2, __dmul_rn(fx, fx)), __dmul_rn(fy, fy));
    if (arg < 0.0) return mk(0.0, 0.0);
    if (p.local && (fabs(fx) > p.fx_lim || fabs(fy) > p.fy_lim)) return mk(0.0, 0.0);
    const double phase = __dmul_rn(p.two_pi_z, sqrt(arg));
    double s, c;
    sincos(phase, &s, &c);
    return mk(c, s);
}

template <>
__device__ __forceinline__ cx<float> tf_value<float>(const TfChan& p, double fx, double fy) {
    const double fx2 = __dmul_rn(fx, fx), fy2 = __dmul_rn(fy, fy);
    const double arg = __dsub_rn(__dsub_rn(p.inv_l2, fx2), fy2);
    if (arg < 0.0) return mk(0.0f, 0.0f);
    if (p.local && (fabs(fx) > p.fx_lim || fabs(fy) > p.fy_lim)) return mk(0.0f, 0.0f);
    const float f2 = static_cast<float>(__dadd_rn(fx2, fy2));
    const float sq = sqrtf(static_cast<float>(arg));
    const float theta = p.phase0 - p.two_pi_z_f * f2 / (p.inv_l + sq);
    float s, c;
    sincosf(theta, &s, &c);
    return mk(c, s);
}

// ---- propagation.cu
FftPlan plan_or_throw(int n);
std::vector<TfChan> make_tf_consts(const holo_wave& wave, const double* z, int L, int w, int h, int local_limit);
template <class T>
void rows_fft(holo_ctx* ctx, const cx<T>* in, cx<T>* out, int n, long long nrows, int dir, T s);
template <class T>
void cols_fft(holo_ctx* ctx, const cx<T>* in, cx<T>* out, int w, int h, int batch, int dir, T s);
// column-pass options: tftab = transfer functions precomputed [L][C][h][w]
// (instead of evaluated per element); [row_lo, row_hi) = the rows that can be
// nonzero on input (col_spectrum) / that are stored (col_replay); -1 = h
template <class T>
struct ColOpts {
    const cx<T>* tftab = nullptr;
    int row_lo = 0, row_hi = -1;
};
template <class T>
void col_spectrum(holo_ctx* ctx, const cx<T>* layers, cx<T>* spec, int w, int h, int C, int L, const TfChan* d_tfc,
                  double pitch, const ColOpts<T>& opt = ColOpts<T>{});
template <class T>
void col_replay(holo_ctx* ctx, const cx<T>* spec, cx<T>* out, int w, int h, int C, int nout, const int* d_plane_of,
                const TfChan* d_tfc, double pitch, const ColOpts<T>& opt = ColOpts<T>{});
void rows_epilogue(holo_ctx* ctx, const cx<float>* in, int w, int h, int C, int nout, int has_holo, cx<float>* holo,
                   cx<float>* replayed, float* intens);
template <class T>
void pad_field(holo_ctx* ctx, const cx<T>* in, cx<T>* out, int w, int h, int C);
template <class T>
void crop_field(holo_ctx* ctx, const cx<T>* in, cx<T>* out, int w, int h, int C);
template <class T>
void accumulate(holo_ctx* ctx, const cx<T>* in, cx<T>* acc, size_t n, bool first);
template <class T>
void intensity(holo_ctx* ctx, const cx<T>* f, T* out, size_t n);
template <class T>
void transfer_function(holo_ctx* ctx, cx<T>* out, int w, int h, int C, const TfChan* d_tfc, double pitch);

// ---- preprocess.cu (f64, compiled without FMA contraction)

// Per-Gaussian record consumed by the compositing kernel (64 bytes).
struct alignas(16) GRec {
    double mu_x, mu_y;        // projected centre, pixels
    float ca, cb, cc;         // -0.5 log2(e) * (inv00, 2 inv01, inv11): g = 2^(ca dx^2 + cb dx dy + cc dy^2)
    float alpha;              // sigmoid(opacity logit)
    float hx;                 // half-extents of the box holding every pixel with a > alpha_floor:
    float col[6];             // amp_c * (cos phi_c, sin phi_c), c < 3
    float hy;                 //   sqrt(F cov_xx), sqrt(F cov_yy), F = 2 ln(alpha / floor); +inf without a floor
};
static_assert(sizeof(GRec) == 64, "GRec must stay 64 bytes");

struct CameraConsts {
    double wc[9];  // world_to_cam, row-major (camera.cpp:16)
    double pos[3];
    double focal, ppx, ppy;
};

struct PreOut {
    GRec* rec;
    int4* rect;              // tile span [x0, x1) x [y0, y1)
    unsigned* count;         // entries per Gaussian
    double* zc;              // depth key
    int* plane;              // hard assignment (argmax)
    unsigned long long* pmask;  // planes passing the gate (soft mode)
    double* rho;             // N x L plane weights (may be null in hard mode)
    unsigned char* touched;  // count > 0
    holo_projected* projected;  // optional full f64 record
    unsigned* flags;         // bit0 degenerate quaternion, bit1 negative amplitude
    unsigned* num_valid;
    // Hard assignment: preprocess also counts the entries per bucket of planes
    // [pb, pe).  A Gaussian with at most kSlots entries takes its in-bucket slots
    // there (atomic with return on bcount, stored in slots[k][N]); larger ones only
    // count into bbig and take slots bcount[b] + (0..bbig[b]) at emission.
    unsigned* slots;         // null: counting left to k_bucket_count (soft mode)
    unsigned* bcount;
    unsigned* bbig;
    int pb, pe, num_tiles;
};
constexpr int kSlots = 8;

void host_world_to_cam(const holo_camera& cam, double wc[9]);
void preprocess(holo_ctx* ctx, const CameraConsts& cc, const holo_raster_settings& st, double near_clip, int L,
                int tiles_x, int tiles_y, const PreOut& out);

constexpr int kSortCap = 1024;     // largest bucket the compositing CTA sorts in shared memory
constexpr int kWarpSortCap = 256;  // buckets up to this size are sorted one warp each (k_sort_small)

// ---- binning.cu
// out = exclusive scan of in (+ in2 when given), out[n] = total; *d_max = max element
void exclusive_scan_u32(holo_ctx* ctx, const unsigned* in, unsigned* out, long long n, unsigned* d_max,
                        const unsigned* in2 = nullptr);
void bucket_count(holo_ctx* ctx, const PreOut& pre, size_t N, int L, int plane_begin, int plane_end, int tiles_x,
                  int num_tiles, int soft, unsigned* bcount);
// validation / status flags written by the frame's kernels (misc[0])
constexpr unsigned kFlagDegenerateQuat = 1u, kFlagNegativeAmp = 2u, kFlagOverflow = 4u;
void bucket_emit(holo_ctx* ctx, const PreOut& pre, size_t N, int L, int plane_begin, int plane_end, int tiles_x,
                 int num_tiles, int soft, const unsigned* bstart, unsigned* cursor,
                 int* egidx, unsigned capacity, unsigned* flags);
// device-driven: buckets above kSortCap (and, one warp each, those of 129..kWarpSortCap
// entries) are found and sorted without a host round trip; d_nlist[0..1] count them
void sort_large_buckets(holo_ctx* ctx, const unsigned* bstart, long long B, unsigned capacity,
                        const unsigned long long* zkey, int* egidx, unsigned* d_nlist);
// make_target_from_scene's per-plane masks [L][P] (f64 0/1) from layers [L][C][P]
void plane_masks(holo_ctx* ctx, const cx<float>* layers, int L, int C, size_t P, double* masks);
void entry_depths(holo_ctx* ctx, const int* egidx, const double* zc, double* edepth, const unsigned* d_E,
                  unsigned capacity);
// host[0..2] = misc[0..2] (flags, num_valid, max bucket), host[4] = *total (E); host is pinned
void publish_status(holo_ctx* ctx, const unsigned* misc, const unsigned* total, unsigned* host_pinned);

// ---- scene_ops.cu: stable subset of the Gaussians whose hard plane is in [pb, pe)
// (src/dst: positions, rotations, log_scales, amplitudes, opacity, phases, plane
// logits); returns the subset size (synchronises the context stream)
size_t scene_keep_planes(holo_ctx* ctx, const double* const src[7], double* const dst[7], size_t n, int L, int pb,
                         int pe);

// ---- render_static.cu (compile-time FFT plans for the common grid sizes)
enum { kModeFull = 0, kModeSpec = 1, kModeReplay = 2 };
bool static_render_supported(int W, int H);
void static_col_fwd(holo_ctx* ctx, cx<float>* data, int W, int H, int nfields);
// [c0, c0 + nc) restricts a launch to those channels (nc < 0: through C - 1)
void static_col_inv(holo_ctx* ctx, const cx<float>* in, int W, int H, int C, int nout, int has_holo,
                    cx<float>* holo, cx<float>* rep, float* intens, int c0 = 0, int nc = -1);
// outputs of modes FULL / REPLAY: [hologram if has_holo] then planes 0..nrep-1
void static_row(holo_ctx* ctx, int mode, const cx<float>* layers, cx<float>* spec, cx<float>* out, int W, int H,
                int C, int Lloc, int has_holo, int nrep, const TfChan* tfc, double pitch, bool local, int c0 = 0,
                int nc = -1);

// ---- composite.cu
struct CompositeArgs {
    const unsigned* bstart;   // bucket_start for the rendered planes, indexed by local bucket
    const unsigned long long* zkey;  // depth bits per Gaussian (the IEEE bits of zc)
    int* egidx;               // gidx per entry
    const GRec* rec;
    const double* rho;        // soft mode weights or null
    int L, C, W, H, tiles_x, num_tiles, plane_begin, num_buckets;
    int soft, write_lists;
    unsigned capacity;        // entry-buffer size: bucket ranges are clamped to it (overflowed async frames)
    float term_eps, alpha_floor, alpha_clamp;
    int floor_positive;
    cx<float>* layers;        // [planes][C][H][W], plane relative to plane_begin
    float* t_final;           // optional [planes][H][W]
    int* n_contrib;           // optional
    int* e_last;              // with n_contrib: bucket-relative index of the last accepted entry (-1: none)
};
void composite(holo_ctx* ctx, const CompositeArgs& a, int tile);

// ---- brute.cu: brute_force_forward (rasterizer.cpp:265-315), layers [L][C][H][W]
void brute_force(holo_ctx* ctx, const GRec* rec, const int* order, int n_order, const int* plane_of,
                 const double* rho, int L, int C, int W, int H, int tile, bool soft, bool gate_open,
                 float alpha_floor, bool floor_positive, float clamp, cx<float>* layers);

// ---- backward.cu
struct alignas(16) BwdRec {  // per Gaussian: cos / sin of the phases, amplitudes, sigmoid(opacity)
    float cs[6];
    float amp[3];
    float alpha;
    float pad[2];
};
struct RasterBwdArgs {
    const unsigned* bstart;
    const int* egidx;          // bucket-major, depth-sorted (the forward's lists)
    const GRec* rec;
    const BwdRec* brec;
    const double* rho;         // soft mode
    int L, C, W, H, tiles_x, num_tiles, plane_begin, num_buckets;
    int soft;
    unsigned capacity;
    float alpha_floor, alpha_clamp;
    int floor_positive;
    const cx<float>* grad_layers;  // [planes][C][H][W]
    const float* t_final;          // the forward's aux outputs
    const int* n_contrib;
    const int* e_last;  // optional: the forward's last accepted entry per pixel (skips the replay pass)
    const unsigned* goff;          // exclusive scan of the per-Gaussian entry counts
    const int4* rect;
    const unsigned long long* pmask;  // soft mode
    float* egrad;                  // [E][13], Gaussian-major (goff[g] + k-th entry of g)
};
struct GaussBwdArgs {
    size_t n;
    int L, pb, pe, num_tiles, tiles_x, soft;
    unsigned capacity;
    const unsigned* bstart;
    const int* egidx;
    const float* egrad;
    const unsigned* goff;
    const int4* rect;
    const unsigned* count;
    const int* plane;
    const unsigned long long* pmask;
    const double *positions, *rotations, *log_scales, *opacity_logits, *plane_logits;
    CameraConsts cam;
    double near_clip, dilation, alpha_floor, soft_tau, ste_tau;
    holo_scene_grads g;
};
void bwd_seed(holo_ctx* ctx, const cx<float>* rep, const float* gi, const double* gi64, cx<float>* gv, size_t n);
void bwd_prep(holo_ctx* ctx, size_t N, const double* amplitudes, const double* phases, const GRec* rec,
              BwdRec* out);
void raster_backward_entries(holo_ctx* ctx, const RasterBwdArgs& a, int tile);
void gauss_backward(holo_ctx* ctx, const GaussBwdArgs& a);
// (zc, gidx) order for buckets of 2..kWarpSortCap entries, written back to egidx
void sort_small_buckets(holo_ctx* ctx, const unsigned* bstart, long long B, unsigned capacity,
                        const unsigned long long* zkey, int* egidx, unsigned* d_nlist);

// ---- training step (training.cu): losses, opacity decay, optimizer
void losses_gpu(holo_ctx* ctx, const double* I, const double* G, const double* masks, int L, int C, int H, int W,
                bool plain, bool with_ssim, double lambda_ssim, double* grad, double* d_out);
void ssim_gpu(holo_ctx* ctx, const double* I, const double* G, int L, int C, int H, int W, double gscale,
              double* grad, double* d_mean);
double opacity_term(holo_ctx* ctx, const double* logits, size_t n, double lambda, double* gopac);

// ---- phase-only conversion (phase_only.cu), f64 fields; "padded" = the 2w x 2h
// grid of pad2x with the w x h field centred (propagation.cpp:64-82)
// e^{j theta} [C][h][w] into the (padded) grid, zeros around it
void phase_field(holo_ctx* ctx, const double* theta, cx<double>* out, int w, int h, int C, bool pad);
// per plane: sum |rep - tf|^2 over the crop (deterministic), images = |rep|^2 [L][C][h][w]
void phase_match(holo_ctx* ctx, const cx<double>* rep, const cx<double>* tf, int w, int h, int C, int L, bool pad,
                 double* images, double* plane_sums);
// in place over rep: gv = 2 inv_lm (rep - tf) + 2 rep gi on the crop, 0 around it
void phase_seed(holo_ctx* ctx, cx<double>* rep, const cx<double>* tf, const double* gi, int w, int h, int C, int L,
                bool pad, double inv_lm);
// grad = Im(acc conj(e^{j theta})) over the crop of acc
void phase_grad(holo_ctx* ctx, const cx<double>* acc, const double* theta, double* grad, int w, int h, int C,
                bool pad);
void phase_arg(holo_ctx* ctx, const cx<double>* P, double* theta, size_t n);
bool all_finite_c128(holo_ctx* ctx, const cx<double>* P, size_t n);
void f32_to_f64(holo_ctx* ctx, const float* in, double* out, size_t n);
void f64_to_f32(holo_ctx* ctx, const double* in, float* out, size_t n);
void replay_intensity_f64(holo_ctx* ctx, const cx<float>* rep, double* out, size_t n);
bool grads_finite(holo_ctx* ctx, const double* const* g, const size_t* n, int groups);
void adaptive_update(holo_ctx* ctx, double* p, const double* g, double* m, double* v, double* nn, double* prev,
                     size_t n, double lr, long long step, double b1, double b2, double b3, double eps, bool adam);
void renormalize_scene(holo_ctx* ctx, double* rot, double* amp, size_t n);

}  // namespace holo_cuda
