/* holo_oracle — plain-C restatement of the reference forward render path.
 *
 * TEST INFRASTRUCTURE (see holo_oracle.h).  Every function names the reference
 * lines it restates.  Arithmetic follows the reference's expression order with
 * FP contraction disabled (built with -ffp-contract=off); 3x3 products use the
 * left-to-right inner-product order documented in oracle/shim/Eigen/Dense, the
 * same order the CUDA preprocessing kernel uses, so projections, tile spans
 * and bucket lists agree bit for bit.
 */
#define _POSIX_C_SOURCE 200809L
#include "holo_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "fft64.h"

static const double kPi = 3.141592653589793;
static const double kTwoPi = 2.0 * 3.141592653589793;

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* ho_last_error(void) { return g_err; }

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* WaveConfig defaults, wave_config.hpp:11-23 */
void ho_default_wave(ho_wave* w) {
    memset(w, 0, sizeof *w);
    w->nx = 128;
    w->ny = 128;
    w->pitch = 3.74e-6;
    w->channels = 3;
    w->wavelengths[0] = 639e-9;
    w->wavelengths[1] = 532e-9;
    w->wavelengths[2] = 473e-9;
    w->distance = 2e-3;
    w->volume_depth = 4e-3;
    w->num_planes = 2;
}

/* CameraView defaults, camera.hpp:14-30 */
void ho_default_camera(ho_camera* c) {
    memset(c, 0, sizeof *c);
    c->focal_px = 150.0;
    c->cx = -1.0;
    c->cy = -1.0;
}

/* RenderSettings defaults, rasterizer.hpp:12-28 */
void ho_default_settings(ho_settings* s) {
    s->near_clip = 0.0;
    s->dilation = 0.3;
    s->plane_eps = 0.5;
    s->term_eps = 1e-4;
    s->alpha_floor = 1.0 / 255.0;
    s->alpha_clamp = 0.999;
    s->radius_form_cap = 0.0;
    s->ste_tau = 1e-3;
    s->soft_assignment = 0;
    s->soft_tau = 1.0;
    s->tile = 16;
}

/* WaveConfig::validate, wave_config.cpp:5-16 */
int ho_wave_validate(const ho_wave* w) {
    if (w->nx <= 0 || w->ny <= 0) return fail(HO_ERR_CONFIG, "resolution must be positive");
    if (w->pitch <= 0.0) return fail(HO_ERR_CONFIG, "pixel pitch must be positive");
    if (w->channels < 1) return fail(HO_ERR_CONFIG, "at least one wavelength required");
    if (w->channels > HO_MAX_CHANNELS) return fail(HO_ERR_CONFIG, "too many wavelength channels");
    for (int c = 0; c < w->channels; ++c)
        if (w->wavelengths[c] <= 0.0) return fail(HO_ERR_CONFIG, "wavelengths must be positive");
    if (w->distance <= 0.0) return fail(HO_ERR_CONFIG, "propagation distance must be positive");
    if (w->volume_depth < 0.0) return fail(HO_ERR_CONFIG, "volume depth must be non-negative");
    if (w->num_planes < 1) return fail(HO_ERR_CONFIG, "need at least one depth plane");
    if (w->num_planes > 1 && w->volume_depth <= 0.0)
        return fail(HO_ERR_CONFIG, "multiple planes need a positive volume depth");
    return HO_OK;
}

/* plane_positions, wave_config.cpp:18-30 */
int ho_plane_positions(const ho_wave* w, double* z) {
    int rc = ho_wave_validate(w);
    if (rc) return rc;
    const int L = w->num_planes;
    if (L == 1) {
        z[0] = w->distance;
        return HO_OK;
    }
    const double dz = w->volume_depth / (L - 1);
    const double z0 = w->distance - 0.5 * (L - 1) * dz;
    for (int l = 0; l < L; ++l) z[l] = z0 + l * dz;
    return HO_OK;
}

/* c = a * b for row-major 3x3, coefficient = left-to-right inner sum */
static void mat3_mul(const double* a, const double* b, double* c) {
    double t[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            t[i * 3 + j] = (a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j]) + a[i * 3 + 2] * b[2 * 3 + j];
    memcpy(c, t, sizeof t);
}

/* rot_cam_to_world = Rz Ry Rx (camera.cpp:5-14); world_to_cam = its transpose (:16) */
void ho_rot_world_to_cam(const ho_camera* c, double wc[9]) {
    const double cx = cos(c->pose[3]), sx = sin(c->pose[3]);
    const double cy = cos(c->pose[4]), sy = sin(c->pose[4]);
    const double cz = cos(c->pose[5]), sz = sin(c->pose[5]);
    const double rx[9] = {1, 0, 0, 0, cx, -sx, 0, sx, cx};
    const double ry[9] = {cy, 0, sy, 0, 1, 0, -sy, 0, cy};
    const double rz[9] = {cz, -sz, 0, sz, cz, 0, 0, 0, 1};
    double t[9], r[9];
    mat3_mul(rz, ry, t);
    mat3_mul(t, rx, r);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) wc[i * 3 + j] = r[j * 3 + i];
}

/* quat_to_rot (scene.cpp:74-82), covariance_3d (scene.cpp:125-130); row-major */
void ho_covariance_3d(const double* q, const double* ls, double sigma[9]) {
    const double norm = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
    const double w = q[0] / norm, x = q[1] / norm, y = q[2] / norm, z = q[3] / norm;
    const double r[9] = {
        1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z),       2.0 * (x * z + w * y),
        2.0 * (x * y + w * z),       1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
        2.0 * (x * z - w * y),       2.0 * (y * z + w * x),       1.0 - 2.0 * (x * x + y * y),
    };
    double m[9];
    for (int k = 0; k < 3; ++k) {
        const double e = exp(ls[k]);
        for (int i = 0; i < 3; ++i) m[i * 3 + k] = r[i * 3 + k] * e;
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            sigma[i * 3 + j] = (m[i * 3 + 0] * m[j * 3 + 0] + m[i * 3 + 1] * m[j * 3 + 1]) + m[i * 3 + 2] * m[j * 3 + 2];
}

/* sigmoid, common.hpp:32-40 */
static double sigmoid(double x) {
    if (x >= 0.0) {
        const double e = exp(-x);
        return 1.0 / (1.0 + e);
    }
    const double e = exp(x);
    return e / (1.0 + e);
}

/* ste_assign forward: argmax, ties to the lowest index (scene.cpp:138-142) */
int ho_ste_argmax(const double* logits, int L) {
    int best = 0;
    for (int l = 1; l < L; ++l)
        if (logits[l] > logits[best]) best = l;
    return best;
}

/* softmax(logits / tau), shifted by the argmax logit (scene.cpp:144-151) */
static void ste_softmax(const double* logits, int L, double tau, double* out) {
    const int best = ho_ste_argmax(logits, L);
    const double top = logits[best];
    double denom = 0.0;
    for (int l = 0; l < L; ++l) {
        out[l] = exp((logits[l] - top) / tau);
        denom += out[l];
    }
    for (int l = 0; l < L; ++l) out[l] /= denom;
}

static double effective_near(const ho_settings* st, const ho_wave* cfg) {
    return st->near_clip > 0.0 ? st->near_clip : 0.2 * cfg->distance; /* rasterizer.hpp:25-27 */
}

/* detail::project_gaussian, rasterizer.cpp:10-70 */
void ho_project(const ho_scene* s, size_t n, const ho_camera* cam, const double wc[9], const ho_wave* cfg,
                const ho_settings* st, ho_projected* p) {
    memset(p, 0, sizeof *p);
    p->n = (int)n;
    const double* xw = s->positions + 3 * n;
    const double d[3] = {xw[0] - cam->pose[0], xw[1] - cam->pose[1], xw[2] - cam->pose[2]};
    double xc[3];
    for (int i = 0; i < 3; ++i) xc[i] = (wc[i * 3 + 0] * d[0] + wc[i * 3 + 1] * d[1]) + wc[i * 3 + 2] * d[2];
    if (!(xc[2] > effective_near(st, cfg))) return;
    p->xc = xc[0];
    p->yc = xc[1];
    p->zc = xc[2];

    const double f = cam->focal_px;
    const double iz = 1.0 / xc[2];
    const double ppx = cam->cx >= 0.0 ? cam->cx : cam->width / 2.0;
    const double ppy = cam->cy >= 0.0 ? cam->cy : cam->height / 2.0;
    p->mu_x = f * xc[0] * iz + ppx;
    p->mu_y = f * xc[1] * iz + ppy;

    /* J = d(pixel)/d(camera point), 2x3 row-major, zeros kept in the products */
    double J[6] = {0, 0, 0, 0, 0, 0};
    J[0] = f * iz;
    J[4] = f * iz;
    J[2] = -f * xc[0] * iz * iz;
    J[5] = -f * xc[1] * iz * iz;

    double sigma[9];
    ho_covariance_3d(s->rotations + 4 * n, s->log_scales + 3 * n, sigma);
    double M[6], T[6], cov[4];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            M[i * 3 + j] = (J[i * 3 + 0] * wc[0 * 3 + j] + J[i * 3 + 1] * wc[1 * 3 + j]) + J[i * 3 + 2] * wc[2 * 3 + j];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            T[i * 3 + j] =
                (M[i * 3 + 0] * sigma[0 * 3 + j] + M[i * 3 + 1] * sigma[1 * 3 + j]) + M[i * 3 + 2] * sigma[2 * 3 + j];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            cov[i * 2 + j] = (T[i * 3 + 0] * M[j * 3 + 0] + T[i * 3 + 1] * M[j * 3 + 1]) + T[i * 3 + 2] * M[j * 3 + 2];
    cov[0] += st->dilation;
    cov[3] += st->dilation;

    const double det = cov[0] * cov[3] - cov[1] * cov[1];
    if (!(det > 0.0) || !isfinite(det)) return;
    const double idet = 1.0 / det;
    p->inv00 = cov[3] * idet;
    p->inv01 = -cov[1] * idet;
    p->inv11 = cov[0] * idet;

    p->alpha_sig = sigmoid(s->opacity_logits[n]);
    if (st->alpha_floor > 0.0 && !(p->alpha_sig > st->alpha_floor)) return;

    double form_cap = st->radius_form_cap;
    if (form_cap <= 0.0) {
        form_cap = 9.0;
        if (st->alpha_floor > 0.0) {
            const double c2 = 2.0 * log(p->alpha_sig / st->alpha_floor);
            form_cap = form_cap < c2 ? c2 : form_cap; /* std::max(9, ..) */
        }
    }
    const double mid = 0.5 * (cov[0] + cov[3]);
    const double disc = mid * mid - det;
    const double lambda_max = mid + sqrt(disc > 0.0 ? disc : 0.0);
    p->radius = sqrt(form_cap * lambda_max);
    for (int ch = 0; ch < 3; ++ch) {
        p->amp[ch] = s->amplitudes[3 * n + ch];
        p->phase[ch] = s->phases[3 * n + ch];
    }
    p->valid = 1;
}

/* GaussianScene::validate (scene.cpp:19-32) */
static int scene_validate(const ho_scene* s) {
    if (s->num_planes < 1) return fail(HO_ERR_CONFIG, "scene needs at least one plane");
    for (size_t i = 0; i < s->n; ++i) {
        const double* q = s->rotations + 4 * i;
        const double norm = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
        if (!(norm > 1e-8)) return fail(HO_ERR_CONFIG, "degenerate quaternion in scene");
    }
    for (size_t i = 0; i < 3 * s->n; ++i)
        if (s->amplitudes[i] < 0.0) return fail(HO_ERR_CONFIG, "amplitudes must be non-negative");
    return HO_OK;
}

/* CameraView::validate (camera.cpp:22-27) */
static int camera_validate(const ho_camera* c) {
    if (c->width <= 0 || c->height <= 0) return fail(HO_ERR_CONFIG, "camera resolution must be positive");
    if (c->focal_px <= 0.0) return fail(HO_ERR_CONFIG, "focal length must be positive");
    for (int i = 0; i < 6; ++i)
        if (!isfinite(c->pose[i])) return fail(HO_ERR_CONFIG, "camera pose must be finite");
    return HO_OK;
}

/* tile_span, rasterizer.cpp:106-113 */
static void tile_span(const ho_projected* p, int tile, int tx, int ty, int span[4]) {
    int x0 = (int)floor((p->mu_x - p->radius) / tile);
    int x1 = (int)floor((p->mu_x + p->radius) / tile) + 1;
    int y0 = (int)floor((p->mu_y - p->radius) / tile);
    int y1 = (int)floor((p->mu_y + p->radius) / tile) + 1;
    span[0] = x0 > 0 ? x0 : 0;
    span[1] = x1 < tx ? x1 : tx;
    span[2] = y0 > 0 ? y0 : 0;
    span[3] = y1 < ty ? y1 : ty;
}

/* evaluate, rasterizer.cpp:124-135; returns accept, fills alpha */
static int evaluate(const ho_projected* p, double rho, double px, double py, const ho_settings* st,
                    double* alpha) {
    const double dx = px - p->mu_x;
    const double dy = py - p->mu_y;
    const double form = p->inv00 * dx * dx + 2.0 * p->inv01 * dx * dy + p->inv11 * dy * dy;
    const double g = exp(-0.5 * form);
    double a = p->alpha_sig * g * rho;
    if (a > st->alpha_clamp) a = st->alpha_clamp;
    *alpha = a;
    return (a > st->alpha_floor) || (st->alpha_floor <= 0.0 && a > 0.0);
}

typedef struct {
    double depth;
    int32_t gidx;
} sort_key;

static int cmp_key(const void* a, const void* b) {
    const sort_key* x = (const sort_key*)a;
    const sort_key* y = (const sort_key*)b;
    if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
    return (x->gidx > y->gidx) - (x->gidx < y->gidx);
}

void ho_raster_free(ho_raster* r) {
    if (!r) return;
    free(r->layers);
    free(r->t_final);
    free(r->n_contrib);
    free(r->projected);
    free(r->rho);
    free(r->touched);
    free(r->entry_bucket);
    free(r->entry_gidx);
    free(r->entry_depth);
    free(r->bucket_start);
    memset(r, 0, sizeof *r);
}

/* Shared front half of raster_forward / brute_force_forward: projection and
 * plane weights (rasterizer.cpp:165-171, compute_rho :81-99). */
static void project_all(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                        ho_projected* proj, double* rho) {
    double wc[9];
    ho_rot_world_to_cam(cam, wc);
    const int L = s->num_planes;
    const long long N = (long long)s->n;
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < N; ++i) {
        ho_project(s, (size_t)i, cam, wc, cfg, st, &proj[i]);
        const double* lg = s->plane_logits + (size_t)i * L;
        double* r = rho + (size_t)i * L;
        for (int l = 0; l < L; ++l) r[l] = 0.0;
        const int best = ho_ste_argmax(lg, L);
        if (st->soft_assignment) {
            ste_softmax(lg, L, st->soft_tau, r);
        } else {
            r[best] = 1.0;
        }
        proj[i].plane = best;
    }
}

/* raster_forward, rasterizer.cpp:139-263 */
int ho_raster_forward(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                      ho_raster* out) {
    memset(out, 0, sizeof *out);
    int rc;
    if ((rc = scene_validate(s))) return rc;
    if ((rc = camera_validate(cam))) return rc;
    if ((rc = ho_wave_validate(cfg))) return rc;
    if (s->num_planes != cfg->num_planes)
        return fail(HO_ERR_CONFIG, "scene plane count does not match the wave config");
    if (cam->width != cfg->nx || cam->height != cfg->ny)
        return fail(HO_ERR_CONFIG, "camera resolution must match the hologram grid");

    const int L = cfg->num_planes, W = cfg->nx, H = cfg->ny, tile = st->tile;
    const size_t N = s->n;
    out->L = L;
    out->w = W;
    out->h = H;
    out->tiles_x = (W + tile - 1) / tile;
    out->tiles_y = (H + tile - 1) / tile;
    const int num_tiles = out->tiles_x * out->tiles_y;
    const size_t P = (size_t)W * H;

    out->layers = (double*)calloc((size_t)L * 3 * P * 2, sizeof(double));
    out->t_final = (double*)malloc(sizeof(double) * (size_t)L * P);
    out->n_contrib = (int32_t*)calloc((size_t)L * P, sizeof(int32_t));
    out->projected = (ho_projected*)calloc(N ? N : 1, sizeof(ho_projected));
    out->rho = (double*)calloc(N * L + 1, sizeof(double));
    out->touched = (uint8_t*)calloc(N ? N : 1, 1);
    for (size_t i = 0; i < (size_t)L * P; ++i) out->t_final[i] = 1.0;

    project_all(s, cam, cfg, st, out->projected, out->rho);

    /* emission counts and prefix sum (:173-187) */
    const double gate = st->soft_assignment ? 0.0 : st->plane_eps;
    uint32_t* emit = (uint32_t*)calloc(N + 1, sizeof(uint32_t));
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < (long long)N; ++i) {
        const ho_projected* p = &out->projected[i];
        if (!p->valid) continue;
        int sp[4];
        tile_span(p, tile, out->tiles_x, out->tiles_y, sp);
        if (sp[0] >= sp[1] || sp[2] >= sp[3]) continue;
        uint32_t planes = 0;
        for (int l = 0; l < L; ++l)
            if (out->rho[(size_t)i * L + l] > gate) ++planes;
        emit[i + 1] = planes * (uint32_t)((sp[1] - sp[0]) * (sp[3] - sp[2]));
    }
    for (size_t i = 0; i < N; ++i) emit[i + 1] += emit[i];
    const size_t E = emit[N];
    out->num_entries = E;

    /* fill in (i, l, ty, tx) order (:188-204) */
    int32_t* eb = (int32_t*)malloc(sizeof(int32_t) * (E ? E : 1));
    int32_t* eg = (int32_t*)malloc(sizeof(int32_t) * (E ? E : 1));
    double* ed = (double*)malloc(sizeof(double) * (E ? E : 1));
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < (long long)N; ++i) {
        uint32_t at = emit[i];
        if (emit[i + 1] == at) continue;
        const ho_projected* p = &out->projected[i];
        int sp[4];
        tile_span(p, tile, out->tiles_x, out->tiles_y, sp);
        out->touched[i] = 1;
        for (int l = 0; l < L; ++l) {
            if (!(out->rho[(size_t)i * L + l] > gate)) continue;
            for (int ty = sp[2]; ty < sp[3]; ++ty)
                for (int tx = sp[0]; tx < sp[1]; ++tx) {
                    eb[at] = l * num_tiles + ty * out->tiles_x + tx;
                    eg[at] = (int32_t)i;
                    ed[at] = p->zc;
                    ++at;
                }
        }
    }
    free(emit);

    /* stable counting sort by bucket, then (depth, gidx) within each bucket (:206-225) */
    const int B = L * num_tiles;
    out->bucket_start = (uint32_t*)calloc((size_t)B + 1, sizeof(uint32_t));
    for (size_t e = 0; e < E; ++e) ++out->bucket_start[eb[e] + 1];
    for (int b = 0; b < B; ++b) out->bucket_start[b + 1] += out->bucket_start[b];
    sort_key* keys = (sort_key*)malloc(sizeof(sort_key) * (E ? E : 1));
    {
        uint32_t* cursor = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)B + 1));
        memcpy(cursor, out->bucket_start, sizeof(uint32_t) * (size_t)B);
        for (size_t e = 0; e < E; ++e) {
            const uint32_t at = cursor[eb[e]]++;
            keys[at].depth = ed[e];
            keys[at].gidx = eg[e];
        }
        free(cursor);
    }
#pragma omp parallel for schedule(dynamic, 8)
    for (int b = 0; b < B; ++b) {
        const uint32_t e0 = out->bucket_start[b], e1 = out->bucket_start[b + 1];
        if (e1 - e0 > 1) qsort(keys + e0, e1 - e0, sizeof(sort_key), cmp_key);
    }
    for (int b = 0; b < B; ++b)
        for (uint32_t e = out->bucket_start[b]; e < out->bucket_start[b + 1]; ++e) {
            eb[e] = b;
            eg[e] = keys[e].gidx;
            ed[e] = keys[e].depth;
        }
    free(keys);
    out->entry_bucket = eb;
    out->entry_gidx = eg;
    out->entry_depth = ed;

    /* front-to-back compositing per (plane, tile) bucket (:227-261) */
#pragma omp parallel for schedule(dynamic, 4)
    for (int b = 0; b < B; ++b) {
        const uint32_t e0 = out->bucket_start[b], e1 = out->bucket_start[b + 1];
        if (e0 == e1) continue;
        const int plane = b / num_tiles;
        const int t = b % num_tiles;
        const int px0 = (t % out->tiles_x) * tile, py0 = (t / out->tiles_x) * tile;
        const int px1 = px0 + tile < W ? px0 + tile : W;
        const int py1 = py0 + tile < H ? py0 + tile : H;
        double* canvas = out->layers + (size_t)plane * 3 * P * 2;
        for (int py = py0; py < py1; ++py) {
            for (int px = px0; px < px1; ++px) {
                const double sx = px + 0.5, sy = py + 0.5;
                double T = 1.0;
                int32_t contrib = 0;
                double acc[3][2] = {{0, 0}, {0, 0}, {0, 0}};
                for (uint32_t e = e0; e < e1; ++e) {
                    if (T < st->term_eps) break;
                    const ho_projected* p = &out->projected[eg[e]];
                    double a;
                    if (!evaluate(p, out->rho[(size_t)p->n * L + plane], sx, sy, st, &a)) continue;
                    const double w = a * T;
                    for (int ch = 0; ch < 3; ++ch) {
                        acc[ch][0] += p->amp[ch] * w * cos(p->phase[ch]);
                        acc[ch][1] += p->amp[ch] * w * sin(p->phase[ch]);
                    }
                    T *= 1.0 - a;
                    ++contrib;
                }
                const size_t ai = ((size_t)plane * H + py) * W + px;
                out->t_final[ai] = T;
                out->n_contrib[ai] = contrib;
                for (int ch = 0; ch < 3; ++ch) {
                    const size_t o = ((size_t)ch * H + py) * W + px;
                    canvas[2 * o] = acc[ch][0];
                    canvas[2 * o + 1] = acc[ch][1];
                }
            }
        }
    }
    return HO_OK;
}

/* brute_force_forward, rasterizer.cpp:265-315 */
typedef struct {
    double zc;
    int idx;
} order_key;

static int cmp_order(const void* a, const void* b) {
    const order_key* x = (const order_key*)a;
    const order_key* y = (const order_key*)b;
    if (x->zc != y->zc) return x->zc < y->zc ? -1 : 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

int ho_brute_force_forward(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                           double* layers) {
    int rc;
    if ((rc = scene_validate(s))) return rc;
    if ((rc = camera_validate(cam))) return rc;
    if ((rc = ho_wave_validate(cfg))) return rc;
    const int L = cfg->num_planes, W = cfg->nx, H = cfg->ny;
    const size_t N = s->n, P = (size_t)W * H;
    ho_projected* proj = (ho_projected*)calloc(N ? N : 1, sizeof(ho_projected));
    double* rho = (double*)calloc(N * s->num_planes + 1, sizeof(double));
    project_all(s, cam, cfg, st, proj, rho);
    order_key* order = (order_key*)malloc(sizeof(order_key) * (N ? N : 1));
    size_t nv = 0;
    for (size_t i = 0; i < N; ++i)
        if (proj[i].valid) {
            order[nv].zc = proj[i].zc;
            order[nv].idx = (int)i;
            ++nv;
        }
    qsort(order, nv, sizeof(order_key), cmp_order);
    memset(layers, 0, sizeof(double) * (size_t)L * 3 * P * 2);
    const double gate = st->soft_assignment ? 0.0 : st->plane_eps;
    const int Ls = s->num_planes;
    for (int plane = 0; plane < L; ++plane) {
        double* canvas = layers + (size_t)plane * 3 * P * 2;
#pragma omp parallel for schedule(static)
        for (int py = 0; py < H; ++py) {
            for (int px = 0; px < W; ++px) {
                const double sx = px + 0.5, sy = py + 0.5;
                double T = 1.0;
                double acc[3][2] = {{0, 0}, {0, 0}, {0, 0}};
                for (size_t k = 0; k < nv; ++k) {
                    const ho_projected* p = &proj[order[k].idx];
                    const double rv = rho[(size_t)p->n * Ls + plane];
                    if (!(rv > gate)) continue;
                    double a;
                    if (!evaluate(p, rv, sx, sy, st, &a)) continue;
                    const double w = a * T;
                    for (int ch = 0; ch < 3; ++ch) {
                        acc[ch][0] += p->amp[ch] * w * cos(p->phase[ch]);
                        acc[ch][1] += p->amp[ch] * w * sin(p->phase[ch]);
                    }
                    T *= 1.0 - a;
                }
                for (int ch = 0; ch < 3; ++ch) {
                    const size_t o = ((size_t)ch * H + py) * W + px;
                    canvas[2 * o] = acc[ch][0];
                    canvas[2 * o + 1] = acc[ch][1];
                }
            }
        }
    }
    free(order);
    free(proj);
    free(rho);
    return HO_OK;
}

/* ---------------------------------------------------------------- FFT / propagation */

static void fft2_sign(double* data, int w, int h, int sign) {
    fft64_plan* pw = fft64_plan_new(w);
    fft64_plan* ph = fft64_plan_new(h);
    fft64_exec_2d(pw, ph, data, w, h, sign);
    fft64_plan_free(pw);
    fft64_plan_free(ph);
}

/* fft2: forward, unnormalised (fft.cpp:33-36) */
void ho_fft2(double* data, int w, int h) { fft2_sign(data, w, h, -1); }

/* ifft2: backward then x 1/(w h) in a separate pass (fft.cpp:38-44) */
void ho_ifft2(double* data, int w, int h) {
    fft2_sign(data, w, h, +1);
    const double s = 1.0 / ((double)w * h);
    const size_t n = (size_t)w * h;
    for (size_t i = 0; i < 2 * n; ++i) data[i] *= s;
}

/* freq_at, propagation.cpp:13-16 */
static double freq_at(int i, int n, double dx) {
    const int k = (i < (n + 1) / 2) ? i : i - n;
    return (double)k / ((double)n * dx);
}

/* build_tf, propagation.cpp:18-54; out C*h*w*2 */
static void build_tf(int w, int h, double pitch, const double* wl, int C, double z, int local_limit, double* out) {
    memset(out, 0, sizeof(double) * 2 * (size_t)w * h * C);
    for (int ch = 0; ch < C; ++ch) {
        const double lambda = wl[ch];
        const double inv_l2 = 1.0 / (lambda * lambda);
        double fx_lim = 0.0, fy_lim = 0.0;
        if (local_limit && z != 0.0) {
            const double du = 1.0 / (w * pitch);
            const double dv = 1.0 / (h * pitch);
            fx_lim = 1.0 / (lambda * sqrt((2.0 * du * z) * (2.0 * du * z) + 1.0));
            fy_lim = 1.0 / (lambda * sqrt((2.0 * dv * z) * (2.0 * dv * z) + 1.0));
        }
        double* base = out + 2 * (size_t)ch * h * w;
#pragma omp parallel for schedule(static)
        for (int y = 0; y < h; ++y) {
            const double fy = freq_at(y, h, pitch);
            double* row = base + 2 * (size_t)y * w;
            for (int x = 0; x < w; ++x) {
                const double fx = freq_at(x, w, pitch);
                const double arg = inv_l2 - fx * fx - fy * fy;
                if (arg < 0.0) continue;
                if (local_limit && z != 0.0 && (fabs(fx) > fx_lim || fabs(fy) > fy_lim)) continue;
                const double phase = kTwoPi * z * sqrt(arg);
                row[2 * x] = cos(phase);
                row[2 * x + 1] = sin(phase);
            }
        }
    }
}

int ho_transfer_function(const ho_wave* cfg, double z, const ho_prop* opt, double* out) {
    int rc = ho_wave_validate(cfg);
    if (rc) return rc;
    const int w = opt && opt->pad2x ? 2 * cfg->nx : cfg->nx;
    const int h = opt && opt->pad2x ? 2 * cfg->ny : cfg->ny;
    build_tf(w, h, cfg->pitch, cfg->wavelengths, cfg->channels, z, opt ? opt->local_band_limit : 0, out);
    return HO_OK;
}

/* apply_tf_channel, propagation.cpp:57-62 */
static void apply_tf_channel(double* data, int w, int h, const double* hz) {
    ho_fft2(data, w, h);
    const size_t n = (size_t)w * h;
    for (size_t i = 0; i < n; ++i) {
        const double a = data[2 * i], b = data[2 * i + 1];
        const double c = hz[2 * i], d = hz[2 * i + 1];
        data[2 * i] = a * c - b * d;
        data[2 * i + 1] = a * d + b * c;
    }
    ho_ifft2(data, w, h);
}

/* propagate, propagation.cpp:93-101 (pad_center/crop_center :64-82) */
int ho_propagate(const double* in, int w, int h, int c, const ho_wave* cfg, double z, const ho_prop* opt,
                 double* out) {
    if (w != cfg->nx || h != cfg->ny || c != cfg->channels)
        return fail(HO_ERR_CONFIG, "propagate: field does not match the configured grid");
    int rc = ho_wave_validate(cfg);
    if (rc) return rc;
    const int pad = opt && opt->pad2x;
    const int ww = pad ? 2 * w : w, hh = pad ? 2 * h : h;
    const size_t pw = (size_t)ww * hh;
    double* tf = (double*)malloc(sizeof(double) * 2 * pw * c);
    build_tf(ww, hh, cfg->pitch, cfg->wavelengths, c, z, opt ? opt->local_band_limit : 0, tf);
    double* work = (double*)calloc(2 * pw * c, sizeof(double));
    const int ox = (ww - w) / 2, oy = (hh - h) / 2;
    for (int ch = 0; ch < c; ++ch)
        for (int y = 0; y < h; ++y)
            memcpy(work + 2 * (((size_t)ch * hh + y + oy) * ww + ox), in + 2 * (((size_t)ch * h + y) * w),
                   sizeof(double) * 2 * w);
#pragma omp parallel for schedule(static)
    for (int ch = 0; ch < c; ++ch) apply_tf_channel(work + 2 * (size_t)ch * pw, ww, hh, tf + 2 * (size_t)ch * pw);
    for (int ch = 0; ch < c; ++ch)
        for (int y = 0; y < h; ++y)
            memcpy(out + 2 * (((size_t)ch * h + y) * w), work + 2 * (((size_t)ch * hh + y + oy) * ww + ox),
                   sizeof(double) * 2 * w);
    free(work);
    free(tf);
    return HO_OK;
}

/* forward_record, propagation.cpp:103-114 */
int ho_forward_record(const double* layers, int L, const ho_wave* cfg, const ho_prop* opt, double* holo) {
    double zs[1024];
    if (cfg->num_planes > 1024) return fail(HO_ERR_CONFIG, "too many planes");
    int rc = ho_plane_positions(cfg, zs);
    if (rc) return rc;
    if (L != cfg->num_planes) return fail(HO_ERR_CONFIG, "forward_record: layer count does not match num_planes");
    const size_t n = (size_t)cfg->nx * cfg->ny * cfg->channels;
    double* p = (double*)malloc(sizeof(double) * 2 * n);
    memset(holo, 0, sizeof(double) * 2 * n);
    for (int l = 0; l < L; ++l) {
        rc = ho_propagate(layers + 2 * n * l, cfg->nx, cfg->ny, cfg->channels, cfg, zs[l], opt, p);
        if (rc) {
            free(p);
            return rc;
        }
        for (size_t i = 0; i < 2 * n; ++i) holo[i] += p[i];
    }
    free(p);
    return HO_OK;
}

/* inverse_propagate, propagation.cpp:116-123 */
int ho_inverse_propagate(const double* holo, const ho_wave* cfg, const ho_prop* opt, double* replayed) {
    double zs[1024];
    if (cfg->num_planes > 1024) return fail(HO_ERR_CONFIG, "too many planes");
    int rc = ho_plane_positions(cfg, zs);
    if (rc) return rc;
    const size_t n = (size_t)cfg->nx * cfg->ny * cfg->channels;
    for (int l = 0; l < cfg->num_planes; ++l) {
        rc = ho_propagate(holo, cfg->nx, cfg->ny, cfg->channels, cfg, -zs[l], opt, replayed + 2 * n * l);
        if (rc) return rc;
    }
    return HO_OK;
}

/* intensity, field.cpp:5-14 */
void ho_intensity(const double* f, size_t samples, double* out) {
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < (long long)samples; ++i) out[i] = f[2 * i] * f[2 * i] + f[2 * i + 1] * f[2 * i + 1];
}

/* pipeline_forward, pipeline.cpp:20-29 */
int ho_pipeline_forward(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                        const ho_prop* opt, ho_raster* raster, double* hologram, double* replayed,
                        double* intensities, double* stage_seconds) {
    if (cfg->channels > 3) return fail(HO_ERR_CONFIG, "propagate: field does not match the configured grid");
    ho_raster local;
    ho_raster* r = raster ? raster : &local;
    double t0 = now_s();
    int rc = ho_raster_forward(s, cam, cfg, st, r);
    if (rc) return rc;
    double t1 = now_s();
    const int L = cfg->num_planes, C = cfg->channels;
    const size_t P = (size_t)cfg->nx * cfg->ny;
    const size_t n = P * C;
    /* channels [0, C) of every 3-channel layer */
    double* layers = (double*)malloc(sizeof(double) * 2 * n * L);
    for (int l = 0; l < L; ++l)
        memcpy(layers + 2 * n * l, r->layers + 2 * P * 3 * l, sizeof(double) * 2 * n);
    rc = ho_forward_record(layers, L, cfg, opt, hologram);
    free(layers);
    if (rc) {
        if (!raster) ho_raster_free(&local);
        return rc;
    }
    double t2 = now_s();
    double* rep = replayed ? replayed : (double*)malloc(sizeof(double) * 2 * n * L);
    rc = ho_inverse_propagate(hologram, cfg, opt, rep);
    double t3 = now_s();
    if (!rc && intensities) ho_intensity(rep, n * L, intensities);
    double t4 = now_s();
    if (!replayed) free(rep);
    if (!raster) ho_raster_free(&local);
    if (stage_seconds) {
        stage_seconds[0] = t1 - t0;
        stage_seconds[1] = t2 - t1;
        stage_seconds[2] = t3 - t2;
        stage_seconds[3] = t4 - t3;
    }
    return rc;
}

/* psnr, losses.cpp:113-132 (one focal-stack image: c channels of h x w) */
double ho_psnr(const double* a, const double* b, size_t n) {
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double e = a[i] - b[i];
        acc += e * e;
    }
    const double mse = acc / (double)n;
    if (mse <= 0.0) return 99.0;
    const double v = 10.0 * log10(1.0 / mse);
    return v < 99.0 ? v : 99.0;
}

/* keep kPi referenced for readers comparing with common.hpp:15-16 */
double ho_pi(void) { return kPi; }
