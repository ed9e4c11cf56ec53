/* holo_oracle — plain-C restatement of the reference's forward render path.
 *
 * TEST INFRASTRUCTURE.  This is the parity checker for the CUDA path: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * The product (libholo_cuda.so) never links or calls it.
 *
 * Restates, in f64 and in the reference's operation order, holo::pipeline_forward
 * (proj/src/pipeline.cpp:20-29) and everything under it: plane_positions
 * (wave_config.cpp:18-30), the camera rotation (camera.cpp:5-16), covariance_3d
 * (scene.cpp:74-82,125-130), ste_assign (scene.cpp:132-152), project_gaussian
 * (rasterizer.cpp:10-70), raster_forward (rasterizer.cpp:139-263),
 * brute_force_forward (rasterizer.cpp:265-315), the angular-spectrum operators
 * (propagation.cpp:13-123), fft2/ifft2 (fft.cpp:33-44) and intensity (field.cpp:5-14).
 * Pinned against the reference compiled from its own sources (oracle/_ref) by
 * tests/test_oracle_pinning.py and the committed fixtures in tests/golden/.
 *
 * Layouts follow the reference: a field is [C][H][W] complex<double>, stored here
 * as interleaved (re, im) doubles; per-plane arrays are [L][...] back to back.
 */
#ifndef HOLO_ORACLE_H
#define HOLO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { HO_OK = 0, HO_ERR_CONFIG = 1, HO_ERR_IO = 2, HO_ERR_USAGE = 3, HO_ERR_NUMERIC = 4 };
#define HO_MAX_CHANNELS 16

/* WaveConfig, wave_config.hpp:11-23 */
typedef struct {
    int nx, ny;
    double pitch;
    int channels;
    double wavelengths[HO_MAX_CHANNELS];
    double distance;
    double volume_depth;
    int num_planes;
} ho_wave;

/* CameraView, camera.hpp:14-30 */
typedef struct {
    double pose[6]; /* x, y, z, rx, ry, rz */
    double focal_px;
    double cx, cy; /* < 0 -> grid centre */
    int width, height;
} ho_camera;

/* RenderSettings, rasterizer.hpp:12-28 */
typedef struct {
    double near_clip, dilation, plane_eps, term_eps, alpha_floor, alpha_clamp, radius_form_cap, ste_tau;
    int soft_assignment;
    double soft_tau;
    int tile;
} ho_settings;

/* PropagationOptions, propagation.hpp:10-13 */
typedef struct {
    int pad2x;
    int local_band_limit;
} ho_prop;

/* GaussianScene, scene.hpp:18-37 (kChannels = 3) */
typedef struct {
    size_t n;
    int num_planes;
    const double* positions;      /* n*3 */
    const double* rotations;      /* n*4, wxyz */
    const double* log_scales;     /* n*3 */
    const double* amplitudes;     /* n*3 */
    const double* opacity_logits; /* n */
    const double* phases;         /* n*3 */
    const double* plane_logits;   /* n*L */
} ho_scene;

/* detail::Projected, rasterizer.hpp:34-45 */
typedef struct {
    int valid;
    int n;
    double mu_x, mu_y;
    double inv00, inv01, inv11;
    double radius;
    double xc, yc, zc;
    double alpha_sig;
    double amp[3];
    double phase[3];
    int plane;
} ho_projected;

/* RasterForward, rasterizer.hpp:63-73 (layers always carry 3 channels) */
typedef struct {
    int L, w, h, tiles_x, tiles_y;
    size_t num_entries;
    double* layers;         /* L*3*h*w*2 */
    double* t_final;        /* L*h*w */
    int32_t* n_contrib;     /* L*h*w */
    ho_projected* projected; /* N */
    double* rho;            /* N*L */
    uint8_t* touched;       /* N */
    int32_t* entry_bucket;  /* E */
    int32_t* entry_gidx;    /* E */
    double* entry_depth;    /* E */
    uint32_t* bucket_start; /* L*tiles+1 */
} ho_raster;

const char* ho_last_error(void);
void ho_default_wave(ho_wave* w);
void ho_default_camera(ho_camera* c);
void ho_default_settings(ho_settings* s);

int ho_wave_validate(const ho_wave* w);
int ho_plane_positions(const ho_wave* w, double* z_out);
/* world_to_cam as a row-major 3x3, camera.cpp:5-16 */
void ho_rot_world_to_cam(const ho_camera* c, double wc[9]);
/* covariance_3d, scene.cpp:125-130; sigma row-major */
void ho_covariance_3d(const double* quat, const double* log_scales, double sigma[9]);
int ho_ste_argmax(const double* logits, int L);
void ho_project(const ho_scene* s, size_t i, const ho_camera* cam, const double wc[9], const ho_wave* cfg,
                const ho_settings* st, ho_projected* out);

int ho_raster_forward(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                      ho_raster* out);
void ho_raster_free(ho_raster* r);
/* brute_force_forward: layers L*3*h*w*2 */
int ho_brute_force_forward(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                           double* layers);

/* fft.cpp:33-44 */
void ho_fft2(double* data, int w, int h);
void ho_ifft2(double* data, int w, int h);
/* transfer_function, propagation.cpp:86-91; out: C*h'*w'*2 (h', w' doubled when pad2x) */
int ho_transfer_function(const ho_wave* cfg, double z, const ho_prop* opt, double* out);
/* propagate, propagation.cpp:93-101; in/out C*h*w*2 (may alias) */
int ho_propagate(const double* in, int w, int h, int c, const ho_wave* cfg, double z, const ho_prop* opt,
                 double* out);
/* forward_record, propagation.cpp:103-114; layers L*C*h*w*2 -> holo C*h*w*2 */
int ho_forward_record(const double* layers, int L, const ho_wave* cfg, const ho_prop* opt, double* holo);
/* inverse_propagate, propagation.cpp:116-123; holo C*h*w*2 -> replayed L*C*h*w*2 */
int ho_inverse_propagate(const double* holo, const ho_wave* cfg, const ho_prop* opt, double* replayed);
/* intensity, field.cpp:5-14 */
void ho_intensity(const double* field, size_t samples, double* out);

/* pipeline_forward, pipeline.cpp:20-29.  The reference requires cfg->channels == 3
 * (raster layers carry GaussianScene::kChannels = 3, propagation.cpp:94-95 checks);
 * for cfg->channels < 3 the render uses raster channels [0, C) -- the C1 adapter of
 * SURVEY.md 8c.  raster (optional) receives the RasterForward; hologram C*h*w*2,
 * replayed L*C*h*w*2 (optional), intensities L*C*h*w (optional).  stage_seconds
 * (optional, 4 entries) = raster, record, replay, intensity wall times. */
int ho_pipeline_forward(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                        const ho_prop* opt, ho_raster* raster, double* hologram, double* replayed,
                        double* intensities, double* stage_seconds);

/* psnr, losses.cpp:113-132: min(99, 10 log10(1/mse)) over all samples */
double ho_psnr(const double* a, const double* b, size_t n);

#ifdef __cplusplus
}
#endif

#endif
