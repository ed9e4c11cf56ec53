/* holo_cuda.h — C-ABI of libholo_cuda.so, the B200 (sm_100a) forward hologram renderer.
 *
 * This is the drop-in boundary for the reference's render path
 * (the headers under /root/reference/proj/include/holo).  Every entry point names the
 * reference interface it replaces.  Plain C: POD structs, raw pointers and
 * sizes, int status codes, no C++ or torch types.  A context owns one CUDA
 * stream plus its scratch; calls enqueue on that stream.  A context is
 * single-threaded; distinct contexts are independent (reference: value
 * functions, reentrant across threads).
 *
 * Errors: every int-returning call returns HOLO_OK or an error code; the
 * message is in holo_last_error() (thread-local).  Codes 1-4 are the
 * reference's HoloError kinds (proj/include/holo/common.hpp:76-79):
 * config, io, usage, numeric.
 *
 * Device field layout: the reference's planar [C][H][W] (field.hpp:9-21) with
 * complex samples as interleaved (re, im) pairs; per-plane stacks are
 * [L][C][H][W].  HOLO_F32 = float pairs (complex64), HOLO_F64 = double pairs.
 */
#ifndef HOLO_CUDA_H
#define HOLO_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HOLO_CUDA_ABI_VERSION 1

enum holo_status {
    HOLO_OK = 0,
    HOLO_ERR_CONFIG = 1,  /* HoloError("config") */
    HOLO_ERR_IO = 2,      /* HoloError("io") */
    HOLO_ERR_USAGE = 3,   /* HoloError("usage") */
    HOLO_ERR_NUMERIC = 4, /* HoloError("numeric") */
    HOLO_ERR_CUDA = 5,    /* CUDA runtime failure */
    HOLO_ERR_OOM = 6,     /* device allocation failed */
    HOLO_ERR_NCCL = 7     /* collective failure (multi-GPU helpers) */
};

enum holo_dtype { HOLO_F32 = 0, HOLO_F64 = 1 };

#define HOLO_MAX_CHANNELS 16

/* holo::WaveConfig, proj/include/holo/wave_config.hpp:11-23 */
typedef struct {
    int nx, ny;
    double pitch;
    int channels;
    double wavelengths[HOLO_MAX_CHANNELS];
    double distance;
    double volume_depth;
    int num_planes;
} holo_wave;

/* holo::CameraView, proj/include/holo/camera.hpp:14-30 (pose = x, y, z, rx, ry, rz) */
typedef struct {
    double pose[6];
    double focal_px;
    double cx, cy;
    int width, height;
} holo_camera;

/* holo::RenderSettings, proj/include/holo/rasterizer.hpp:12-28 */
typedef struct {
    double near_clip, dilation, plane_eps, term_eps, alpha_floor, alpha_clamp, radius_form_cap, ste_tau;
    int soft_assignment;
    double soft_tau;
    int tile;
} holo_raster_settings;

/* holo::PropagationOptions, proj/include/holo/propagation.hpp:10-13 */
typedef struct {
    int pad2x;
    int local_band_limit;
} holo_prop_options;

/* holo::GaussianScene, proj/include/holo/scene.hpp:18-37: SoA f64, N Gaussians,
 * 3 amplitude/phase channels, num_planes plane logits per Gaussian. */
typedef struct {
    size_t n;
    int num_planes;
    const double* positions;      /* n*3 */
    const double* rotations;      /* n*4 (w, x, y, z) */
    const double* log_scales;     /* n*3 */
    const double* amplitudes;     /* n*3 */
    const double* opacity_logits; /* n */
    const double* phases;         /* n*3 */
    const double* plane_logits;   /* n*num_planes */
} holo_scene_arrays;

/* Outputs of a render (which buffers holo_render fills). */
enum holo_output {
    HOLO_OUT_LAYERS = 1u << 0,    /* RasterForward::layers   [L][C][H][W] complex64 */
    HOLO_OUT_HOLOGRAM = 1u << 1,  /* PipelineForward::hologram [C][H][W] complex64 */
    HOLO_OUT_REPLAYED = 1u << 2,  /* PipelineForward::replayed [L][C][H][W] complex64 */
    HOLO_OUT_INTENSITY = 1u << 3, /* PipelineForward::intensities [L][C][H][W] float32 */
    HOLO_OUT_AUX = 1u << 4,       /* RasterForward::t_final (f32) and n_contrib (i32), [L][H][W] */
    HOLO_OUT_LISTS = 1u << 5,     /* RasterForward::entries / bucket_start */
    HOLO_OUT_PROJECTED = 1u << 6  /* RasterForward::projected (holo_projected, f64) */
};

/* Buffer ids for holo_frame_buffer(). */
enum holo_buffer {
    HOLO_BUF_LAYERS = 0,       /* float2 [L][C][H][W] */
    HOLO_BUF_HOLOGRAM = 1,     /* float2 [C][H][W] */
    HOLO_BUF_REPLAYED = 2,     /* float2 [L][C][H][W] */
    HOLO_BUF_INTENSITY = 3,    /* float [L][C][H][W] */
    HOLO_BUF_T_FINAL = 4,      /* float [L][H][W] */
    HOLO_BUF_N_CONTRIB = 5,    /* int32 [L][H][W] */
    HOLO_BUF_ENTRY_GIDX = 6,   /* int32 [E], bucket-major, depth-sorted (Entry::gidx) */
    HOLO_BUF_ENTRY_DEPTH = 7,  /* double [E] (Entry::depth = camera-space z) */
    HOLO_BUF_BUCKET_START = 8, /* uint32 [B+1] */
    HOLO_BUF_PROJECTED = 9,    /* holo_projected [N] */
    HOLO_BUF_RHO = 10,         /* float [N][L] plane weights used */
    HOLO_BUF_TOUCHED = 11,     /* uint8 [N] */
    HOLO_BUF_SPECTRUM = 12,    /* float2 [C][H][W]: S = sum_l H_{Z_l} FFT2(U_l) (unnormalised) */
    HOLO_BUF_COUNT = 13
};

/* detail::Projected, proj/include/holo/rasterizer.hpp:34-45 */
typedef struct {
    int32_t valid;
    int32_t n;
    double mu_x, mu_y;
    double inv00, inv01, inv11;
    double radius;
    double xc, yc, zc;
    double alpha_sig;
    double amp[3];
    double phase[3];
    int32_t plane;
    int32_t pad_;
} holo_projected;

/* Per-frame facts reported back to the host. */
typedef struct {
    uint64_t num_entries; /* E: (bucket, Gaussian) work items */
    int32_t tiles_x, tiles_y;
    int32_t num_buckets;  /* L * tiles */
    int32_t max_bucket;   /* largest bucket (entries) */
    int32_t num_valid;    /* Gaussians that passed projection culling */
    int32_t pad_;
} holo_frame_info;

typedef struct holo_ctx holo_ctx;

/* ---- context ---- */
const char* holo_last_error(void);
int holo_abi_version(void);
int holo_ctx_create(int device, holo_ctx** out);
int holo_ctx_destroy(holo_ctx* ctx);
/* Enqueue on a caller stream (cudaStream_t cast to void*); NULL is the legacy
 * default stream (what torch.cuda.current_stream() reports as 0). */
int holo_ctx_set_stream(holo_ctx* ctx, void* stream);
/* Back to the context's own non-blocking stream. */
int holo_ctx_use_own_stream(holo_ctx* ctx);
void* holo_ctx_get_stream(holo_ctx* ctx);
/* The context's copy streams (0: host uploads, 1: asynchronous downloads), for
 * callers that order their own work after them. */
void* holo_ctx_get_copy_stream(holo_ctx* ctx, int which);
int holo_ctx_synchronize(holo_ctx* ctx);
/* Optional per-stage CUDA-event timing (ms), accumulated over renders until reset.
 * Stage ids: 0 preprocess, 1 binning, 2 composite, 3 row FFT, 4 column forward,
 * 5 column inverse, 6 row inverse + epilogue. */
int holo_ctx_enable_timing(holo_ctx* ctx, int enable);
int holo_ctx_stage_times(holo_ctx* ctx, double* ms_out, int* launches_out, int max_stages);
int holo_ctx_reset_timing(holo_ctx* ctx);
/* Kernel launches issued by this context since creation. */
uint64_t holo_ctx_launch_count(holo_ctx* ctx);
/* Guard mode (also HOLO_GUARD=1 at creation; set before the first render): scratch
 * buffers get their exact size plus a 4 KB guard band; holo_ctx_check_guards
 * synchronises and reports any band overwritten (HOLO_ERR_NUMERIC, buffer names). */
int holo_ctx_set_guard(holo_ctx* ctx, int enable);
int holo_ctx_check_guards(holo_ctx* ctx);
/* Asynchronous frames.  By default a render makes one host round trip (entry
 * count + scene validation) and returns with its outputs complete, like the
 * reference.  With async enabled a render only enqueues work: the entry buffers
 * hold the reserved capacity (holo_ctx_reserve_entries, or 1.25x the largest
 * synchronous frame so far), the frame info is filled by holo_ctx_frame_status,
 * and validation failures / capacity overflow are reported there (HOLO_ERR_CONFIG /
 * HOLO_ERR_NUMERIC) for every frame since the previous status call.  Renders on
 * one context are stream-ordered; several contexts on separate streams overlap. */
int holo_ctx_set_async(holo_ctx* ctx, int enable);
int holo_ctx_reserve_entries(holo_ctx* ctx, uint64_t entries);
/* Waits for the context's frames, reports the last frame's info and any error
 * flag raised since the previous call (then clears the flags). */
int holo_ctx_frame_status(holo_ctx* ctx, holo_frame_info* info);

/* ---- scene (GaussianScene, scene.hpp:18-37; validated like GaussianScene::validate, scene.cpp:19-32) ---- */
/* Copies host arrays to the device (H2D on the context stream). */
int holo_scene_upload(holo_ctx* ctx, const holo_scene_arrays* host);
/* Copies from device arrays already resident in HBM (D2D). */
int holo_scene_upload_device(holo_ctx* ctx, const holo_scene_arrays* dev);

/* ---- render ----
 * holo_render replaces holo::pipeline_forward (pipeline.cpp:20-29) and, with only
 * raster outputs requested, holo::raster_forward (rasterizer.cpp:139-263).
 * Raster layers carry wave->channels channels: channels [0, C) of the scene's three
 * (C = 3 is the reference; C < 3 is the documented single-wavelength adapter).
 * Outputs live in context-owned device buffers until the next render; fetch them
 * with holo_frame_buffer / holo_frame_download. */
int holo_render(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave, const holo_raster_settings* settings,
                const holo_prop_options* prop, unsigned outputs, holo_frame_info* info);

/* brute_force_forward (rasterizer.hpp:85-86, rasterizer.cpp:265-315): the same
 * per-pixel math as holo_render's tiled raster with no tiles, no support-radius
 * culling and no early termination (every valid Gaussian of a plane, global
 * (depth, index) order, at every pixel) -- the reference's equivalence oracle.
 * Writes HOLO_BUF_LAYERS (the frame's other buffers are those of a raster-only
 * holo_render with HOLO_OUT_PROJECTED). */
int holo_brute_force_forward(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave,
                             const holo_raster_settings* settings);

/* Plane-sharded halves of holo_render (one process per GPU).  begin: rasterise
 * planes [plane_begin, plane_end) and write their partial spectrum
 * S_g = sum_{l in g} H_{Z_l} FFT2(U_l) (float2 [C][H][W]) to spectrum_out
 * (device pointer; NULL = context buffer).  The caller sums S_g over shards
 * (one allreduce) and calls end with the full spectrum to produce the hologram
 * (if HOLO_OUT_HOLOGRAM) and the replayed fields / intensities of planes
 * [plane_begin, plane_end).  Valid only without pad2x. */
int holo_render_begin(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave,
                      const holo_raster_settings* settings, const holo_prop_options* prop, int plane_begin,
                      int plane_end, void* spectrum_out, unsigned outputs, holo_frame_info* info);
int holo_render_end(holo_ctx* ctx, const holo_wave* wave, const holo_prop_options* prop, int plane_begin,
                    int plane_end, const void* spectrum, unsigned outputs);

/* ---- multi-GPU groups: planes, views, planes x views ----
 * The reference has no distributed code.  The unit that is split is
 * one pipeline_forward frame (pipeline.cpp:20-29):
 *   planes  forward_record's sum over planes (propagation.cpp:103-114) is linear,
 *           and hard assignment puts each Gaussian in one plane (rasterizer.cpp:
 *           91-96): a rank renders planes [plane_begin, plane_end) of its plane
 *           group, the partial spectra are summed channel by channel (the sum of
 *           channel c overlaps the row pass of channel c + 1), and the rank forms
 *           its planes' replays / intensities and the hologram channels c with
 *           c mod plane_split == its plane rank.
 *   views   independent frames of one resident scene, as train iterates views
 *           (trainer.cpp:118-133; holo_main.cpp:241-258 --view-index): no
 *           per-frame collective.
 *   both    world = view_groups x plane_split; the sum runs inside each plane
 *           group (ranks r with equal r / plane_split).
 * Mesh: plane_split = ranks per plane group (1 = views only, world = planes only).
 * Views [view_begin, view_end) of a num_views batch go to view group r / plane_split.
 * Transports: NCCL (one process per GPU from a shared unique id, or one process
 * driving several devices), or a caller callback that sums `count` floats of a
 * device buffer over the plane group, ordered on `stream` (tests, custom fabrics). */
typedef struct holo_group holo_group;
#define HOLO_GROUP_ID_BYTES 128

typedef struct {
    int world, rank;
    int plane_split;             /* ranks per plane group */
    int view_groups;             /* world / plane_split */
    int plane_rank, view_group;  /* this rank's coordinates */
    int plane_begin, plane_end;  /* planes this rank renders */
    int view_begin, view_end;    /* views of the batch this rank renders */
    unsigned holo_channels;      /* bit c: this rank forms hologram channel c */
} holo_mesh;

/* Pure host arithmetic (no device): the coordinates above for (world, rank). */
int holo_mesh_layout(int world, int rank, int plane_split, int num_planes, int num_views, int channels,
                     holo_mesh* out);

typedef int (*holo_allreduce_fn)(void* user, float* device_buffer, size_t count, void* cuda_stream);

int holo_group_unique_id(unsigned char id[HOLO_GROUP_ID_BYTES]);
/* one process per GPU: every rank passes the same id (rank 0's, broadcast by the
 * caller); ctx stays the caller's. */
int holo_group_init_rank(holo_ctx* ctx, const unsigned char id[HOLO_GROUP_ID_BYTES], int world, int rank,
                         int plane_split, holo_group** out);
int holo_group_init_callback(holo_ctx* ctx, int world, int rank, int plane_split, holo_allreduce_fn fn, void* user,
                             holo_group** out);
/* one process, n devices (ncclCommInitAll); the group creates and owns a context per device */
int holo_group_create(const int* devices, int n, int plane_split, holo_group** out);
int holo_group_destroy(holo_group* g);
/* local ranks of this process (1, or n for holo_group_create) and their contexts */
int holo_group_local_count(const holo_group* g);
int holo_group_context(holo_group* g, int local, holo_ctx** ctx);
/* frames in flight per local rank (each lane: its own stream and scene copy; default 1) */
int holo_group_set_lanes(holo_group* g, int lanes);
/* upload the full scene on every local rank; a rank of a plane-sharded group keeps
 * its planes' Gaussians only (device-side stable subset). */
int holo_group_upload_scene(holo_group* g, const holo_scene_arrays* host);

/* caller-owned device destinations of one view on one local rank (NULL members:
 * the lane's context buffers).  hologram [C][H][W] complex64 (channels this rank
 * forms); replayed [np][C][H][W] complex64 and intensities [np][C][H][W] float32
 * for the rank's planes. */
typedef struct {
    void* hologram;
    void* replayed;
    void* intensities;
} holo_view_outputs;

enum {
    HOLO_GROUP_GATHER_HOLOGRAM = 1u << 0, /* every rank of a plane group gets all hologram channels */
    HOLO_GROUP_SHARDED_PATH = 1u << 1     /* run the plane-sharded pipeline even for plane groups of one (tests) */
};

/* Render views [view_begin, view_end) of cams[0..num_views) on every local rank.
 * outs / infos: NULL or num_views x local_count entries, index v * local_count + local
 * (only the entries of views a rank renders are used / written). */
int holo_group_render(holo_group* g, const holo_camera* cams, int num_views, const holo_wave* wave,
                      const holo_raster_settings* settings, const holo_prop_options* prop, unsigned outputs,
                      unsigned flags, const holo_view_outputs* outs, holo_frame_info* infos);
int holo_group_synchronize(holo_group* g);
/* holo_ctx_set_async on every lane (the lanes share the largest reservation) */
int holo_group_set_async(holo_group* g, int enable);
/* holo_ctx_frame_status over every lane: the first failure is returned */
int holo_group_frame_status(holo_group* g);
/* make `stream` (a cudaStream_t on local rank's device) wait for all of that
 * rank's work enqueued so far (its lanes and collectives) */
int holo_group_join(holo_group* g, int local, void* stream);
/* kernel launches of all lanes of all local ranks */
uint64_t holo_group_launch_count(const holo_group* g);
/* local rank's mesh coordinates for a batch of num_views views of the wave's planes */
int holo_group_mesh(const holo_group* g, int local, int num_planes, int num_views, int channels, holo_mesh* out);

/* ---- gradients (rasterizer.hpp:79-81 raster_backward; pipeline.cpp:63-91) ----
 * Scene-shaped gradient arrays, device f64 (SceneGradients, scene.hpp:40-46;
 * mu_screen is N x 2).  NULL members are not written; the others are overwritten. */
typedef struct {
    double* positions;      /* n*3 */
    double* rotations;      /* n*4 */
    double* log_scales;     /* n*3 */
    double* amplitudes;     /* n*3 */
    double* opacity_logits; /* n */
    double* phases;         /* n*3 */
    double* plane_logits;   /* n*num_planes */
    double* mu_screen;      /* n*2 */
} holo_scene_grads;

/* raster_backward (rasterizer.cpp:332-528) of the context's last holo_render,
 * which must have requested HOLO_OUT_AUX, on the same camera / wave / settings,
 * with the scene not re-uploaded since.  grad_layers = dL/d(layers): device
 * float2 [L][C][H][W].  Per-entry gradients are fp32 (reduced in a fixed
 * per-warp order, across a tile's warps by shared-memory float atomics); the
 * per-Gaussian merge (entry order, as the reference) and the chain to the
 * parameters are f64. */
int holo_raster_backward(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave,
                         const holo_raster_settings* settings, const void* grad_layers, holo_scene_grads* grads);

/* The gradient branch of total_loss (pipeline.cpp:63-80) for a given
 * dL/d(intensities) (device float [L][C][H][W]): gv_l = 2 replayed_l dL/dI_l, the
 * adjoint of the replay and of the recording (grad_hologram = sum_l propagate(gv_l,
 * +Z_l), grad_layers_l = propagate(grad_hologram, -Z_l): the forward propagation
 * applied to gv), then raster_backward.  Needs the last holo_render with
 * HOLO_OUT_REPLAYED | HOLO_OUT_AUX.  grad_layers_out (float2 [L][C][H][W]) and
 * grad_hologram_out (float2 [C][H][W]) are optional device outputs. */
int holo_pipeline_backward(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave,
                           const holo_raster_settings* settings, const holo_prop_options* prop,
                           const void* grad_intensities, holo_scene_grads* grads, void* grad_layers_out,
                           void* grad_hologram_out);

/* ---- training step: losses (losses.hpp, ssim.hpp), total_loss (pipeline.cpp:30-95),
 * optimizer_step (optimizer.hpp) ---- */
/* PipelineOptions' loss weights (pipeline.hpp:26-28): defaults 0.005, 1e-4, 0. */
typedef struct {
    double lambda_ssim;
    double lambda_opacity;
    int use_plain_mse;
} holo_loss_options;

/* LossBreakdown (pipeline.hpp:44-48); the per-plane PSNR goes to a separate array. */
typedef struct {
    double total, recon, ssim, opacity, psnr_mean;
} holo_loss_breakdown;

/* loss_recon (or loss_mse) + loss_ssim + psnr (losses.cpp) over device f64 focal
 * stacks: intensities / targets [L][C][H][W], masks [L][H][W] (unused by plain MSE).
 * out->opacity = 0; psnr (host, [L]) optional; grad (device f64 [L][C][H][W],
 * optional) receives dL/dI.  f64 throughout; the row sums are folded in the
 * reference's order.  Needs H, W >= 11 (ssim.cpp:71-72) unless lambda_ssim = 0, which
 * leaves the SSIM term out (the loss_mse / loss_recon / psnr of losses.hpp alone). */
int holo_losses(holo_ctx* ctx, const double* intensities, const double* targets, const double* masks, int L, int C,
                int H, int W, const holo_loss_options* opt, holo_loss_breakdown* out, double* psnr, double* grad);

/* total_loss (pipeline.cpp:30-95) on the context's resident scene: render
 * (pipeline_forward), losses against targets / masks (device f64 as above), and
 * with grads != NULL the full gradient (holo_pipeline_backward + the opacity decay
 * term, pipeline.cpp:82-88).  The intensities entering the losses are |replayed|^2
 * in f64 of the fp32 replay (what holo_intensity(HOLO_F64) gives for the widened
 * field).  The frame's outputs stay readable as after holo_render with
 * HOLO_OUT_REPLAYED | HOLO_OUT_AUX. */
int holo_total_loss(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave, const holo_raster_settings* settings,
                    const holo_prop_options* prop, const holo_loss_options* opt, const double* targets,
                    const double* masks, holo_loss_breakdown* out, double* psnr, holo_scene_grads* grads);

/* ssim_mean (ssim.cpp:64-147) of every plane of device f64 stacks [L][C][H][W]:
 * mean_ssim (host, [L]); grad (device, optional) = d(mean SSIM_l)/dx_l, overwritten.
 * Bit-equal to the reference's ssim_mean on the same inputs. */
int holo_ssim(holo_ctx* ctx, const double* x, const double* y, int L, int C, int H, int W, double* mean_ssim,
              double* grad);

/* make_target_from_scene's masks (pipeline.cpp:106-124) of the last frame rendered
 * with HOLO_OUT_LAYERS: masks (device, f64 [num_planes][ny][nx], overwritten) = 1
 * where the plane's sum over channels of |layer| (f64 of the fp32 layer) is the
 * strict maximum over planes (the first on ties), else 0; untouched pixels are 0
 * in every plane. */
int holo_plane_masks(holo_ctx* ctx, double* masks);

/* OptimizerConfig (optimizer.hpp:17-31). */
typedef struct {
    double lr_positions, lr_rotations, lr_log_scales, lr_amplitudes, lr_phases, lr_opacities, lr_plane_logits;
    double beta1, beta2, beta3, eps;
    int use_adam;
    long long schedule_total;
    double lr_floor;
} holo_optimizer_config;

/* OptimState (optimizer.hpp:37-52): device moments, sized at the first step. */
typedef struct holo_optim holo_optim;
int holo_optim_create(holo_ctx* ctx, holo_optim** out);
int holo_optim_destroy(holo_optim* st);
/* optimizer_step (optimizer.cpp:102-133) on the context's resident scene, in place
 * (the arrays the next render reads): *applied = 0 and the skip counted when any
 * gradient entry is non-finite.  grads as from holo_total_loss (all seven groups). */
int holo_optim_step(holo_ctx* ctx, holo_optim* st, const holo_scene_grads* grads, const holo_optimizer_config* cfg,
                    int* applied);
int holo_optim_counts(const holo_optim* st, long long* step, long long* skipped);
/* adaptive_moment_update (optimizer.cpp:70-100) on one flat group of device f64
 * arrays (params, grads, moments m / v / n / prev_grad); step counts from 1.
 * optimizer_step = this per group + the cosine schedule + renormalize. */
int holo_adaptive_update(holo_ctx* ctx, double* params, const double* grads, double* m, double* v, double* n,
                         double* prev_grad, size_t count, double lr, long long step,
                         const holo_optimizer_config* cfg);

/* Copies the resident scene to host arrays (the members are written despite the
 * const qualifiers of holo_scene_arrays; n and num_planes must match). */
int holo_scene_download(holo_ctx* ctx, const holo_scene_arrays* host);

/* ---- phase-only conversion (phase_only.hpp) ----
 * PhaseOnlyOptions (phase_only.hpp:22-32): defaults lambda_ssim 1.0, prop.pad2x 1,
 * use_adam 0.  Fields are device complex128 [C][H][W] (H = wave->ny, W = wave->nx,
 * C = wave->channels), phases device f64 [C][H][W]. */
typedef struct {
    double lambda_ssim;
    holo_prop_options prop;
    int use_adam;
} holo_phase_options;

/* phase_only_loss (phase_only.cpp:104-111): *loss (host) and, when grad != NULL,
 * d loss / d theta (device). */
int holo_phase_only_loss(holo_ctx* ctx, const void* P, const double* theta, const holo_wave* wave,
                         const holo_phase_options* opt, double* loss, double* grad);
/* convert_phase_only (phase_only.cpp:113-160): adaptive-moment descent on theta
 * with the reference's backtracking; phase_out (device) receives the best iterate,
 * trace (host, iters + 1) the loss at initialisation and after every iteration.
 * theta0 (device, optional) is the starting phase; NULL starts from arg(P)
 * computed on the device (the reference's std::arg may differ in the last bit --
 * callers holding P on the host pass their own arg for bit-equal extraction). */
int holo_convert_phase_only(holo_ctx* ctx, const void* P, const holo_wave* wave, int iters, double lr,
                            const holo_phase_options* opt, const double* theta0, double* phase_out, double* trace);

/* Device pointer and size of one output buffer of the last render. */
int holo_frame_buffer(holo_ctx* ctx, int buffer, void** dev_ptr, size_t* bytes);
/* Synchronous device-to-host copy of one output buffer (bytes must match). */
int holo_frame_download(holo_ctx* ctx, int buffer, void* host, size_t bytes);
/* The same copy enqueued on the context stream (pinned host memory overlaps it
 * with other streams' work); complete after holo_ctx_synchronize. */
int holo_frame_download_async(holo_ctx* ctx, int buffer, void* host, size_t bytes);

/* ---- operators on device fields (propagation.hpp:27-40, fft.hpp:11-12, field.hpp:45) ---- */
/* fft2 / ifft2 (fft.cpp:33-44): in place, batch fields of h x w; inverse carries 1/(w h). */
int holo_fft2(holo_ctx* ctx, void* data, int w, int h, int batch, int inverse, int dtype);
/* transfer_function (propagation.cpp:86-91): out [C][h'][w'] (doubled when pad2x). */
int holo_transfer_function(holo_ctx* ctx, const holo_wave* wave, double z, const holo_prop_options* prop,
                           void* out, int dtype);
/* propagate (propagation.cpp:93-101): in/out [C][H][W]; c must equal wave->channels. */
int holo_propagate(holo_ctx* ctx, const void* in, void* out, int w, int h, int c, const holo_wave* wave, double z,
                   const holo_prop_options* prop, int dtype);
/* forward_record (propagation.cpp:103-114): layers [L][C][H][W] -> hologram [C][H][W]. */
int holo_forward_record(holo_ctx* ctx, const void* layers, int num_layers, void* hologram, const holo_wave* wave,
                        const holo_prop_options* prop, int dtype);
/* inverse_propagate (propagation.cpp:116-123): hologram [C][H][W] -> replayed [L][C][H][W]. */
int holo_inverse_propagate(holo_ctx* ctx, const void* hologram, void* replayed, const holo_wave* wave,
                           const holo_prop_options* prop, int dtype);
/* intensity (field.cpp:5-14): |u|^2 per sample; out is float for F32, double for F64. */
int holo_intensity(holo_ctx* ctx, const void* field, void* out, size_t samples, int dtype);
/* f64 intensity of complex64 device samples widened to f64: bitwise the f64 operator
 * applied to the widened field (the drop-in's pipeline_forward intensities equal
 * intensity(replayed) of its returned fields, pipeline.cpp:26-27, test_pipeline.cpp:50-53) */
int holo_intensity_widened(holo_ctx* ctx, const void* field, double* out, size_t samples);

/* Supported FFT lengths: every n whose prime factors are <= 31. */
int holo_fft_supported(int n);

#ifdef __cplusplus
}
#endif

#endif
