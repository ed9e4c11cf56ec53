// ref_capi — extern "C" entry points into the reference library built from
// /root/reference/proj/src by oracle/Makefile (oracle/_ref/libholoref.so).
//
// TEST INFRASTRUCTURE: lets the Python tests and bench.py's reference arm call
// the reference's own C++ functions (holo::pipeline_forward and the operators
// under it) with the plain structs of oracle/holo_oracle.h.  Nothing here
// re-implements the algorithm; it only marshals arguments.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "holo_oracle.h"
#include "holo/fft.hpp"
#include "holo/pipeline.hpp"
#include "holo/propagation.hpp"
#include "holo/rasterizer.hpp"
#include "holo/losses.hpp"
#include "holo/optimizer.hpp"
#include "holo/phase_only.hpp"

namespace {

thread_local std::string g_err;

int code_for(const holo::HoloError& e) {
    if (e.kind == "config") return HO_ERR_CONFIG;
    if (e.kind == "io") return HO_ERR_IO;
    if (e.kind == "usage") return HO_ERR_USAGE;
    return HO_ERR_NUMERIC;
}

holo::WaveConfig to_wave(const ho_wave* w) {
    holo::WaveConfig c;
    c.nx = w->nx;
    c.ny = w->ny;
    c.pitch = w->pitch;
    c.wavelengths.assign(w->wavelengths, w->wavelengths + w->channels);
    c.distance = w->distance;
    c.volume_depth = w->volume_depth;
    c.num_planes = w->num_planes;
    return c;
}

holo::CameraView to_camera(const ho_camera* c) {
    holo::CameraView v;
    for (int i = 0; i < 6; ++i) v.pose[i] = c->pose[i];
    v.focal_px = c->focal_px;
    v.cx = c->cx;
    v.cy = c->cy;
    v.width = c->width;
    v.height = c->height;
    return v;
}

holo::RenderSettings to_settings(const ho_settings* s) {
    holo::RenderSettings r;
    r.near_clip = s->near_clip;
    r.dilation = s->dilation;
    r.plane_eps = s->plane_eps;
    r.term_eps = s->term_eps;
    r.alpha_floor = s->alpha_floor;
    r.alpha_clamp = s->alpha_clamp;
    r.radius_form_cap = s->radius_form_cap;
    r.ste_tau = s->ste_tau;
    r.soft_assignment = s->soft_assignment != 0;
    r.soft_tau = s->soft_tau;
    r.tile = s->tile;
    return r;
}

holo::PropagationOptions to_prop(const ho_prop* p) {
    holo::PropagationOptions o;
    if (p) {
        o.pad2x = p->pad2x != 0;
        o.local_band_limit = p->local_band_limit != 0;
    }
    return o;
}

holo::GaussianScene to_scene(const ho_scene* s) {
    holo::GaussianScene g;
    g.num_planes = s->num_planes;
    const size_t n = s->n;
    g.positions.assign(s->positions, s->positions + 3 * n);
    g.rotations.assign(s->rotations, s->rotations + 4 * n);
    g.log_scales.assign(s->log_scales, s->log_scales + 3 * n);
    g.amplitudes.assign(s->amplitudes, s->amplitudes + 3 * n);
    g.opacity_logits.assign(s->opacity_logits, s->opacity_logits + n);
    g.phases.assign(s->phases, s->phases + 3 * n);
    g.plane_logits.assign(s->plane_logits, s->plane_logits + n * static_cast<size_t>(s->num_planes));
    return g;
}

holo::ComplexField to_field(const double* d, int w, int h, int c, double pitch) {
    holo::ComplexField f(w, h, c, pitch);
    std::memcpy(f.data.data(), d, sizeof(double) * 2 * f.data.size());
    return f;
}

void copy_raster(const holo::RasterForward& r, int L, int w, int h, ho_raster* o) {
    std::memset(o, 0, sizeof *o);
    const size_t P = static_cast<size_t>(w) * h, N = r.projected.size(), E = r.entries.size();
    o->L = L;
    o->w = w;
    o->h = h;
    o->tiles_x = r.tiles_x;
    o->tiles_y = r.tiles_y;
    o->num_entries = E;
    o->layers = static_cast<double*>(std::malloc(sizeof(double) * 2 * 3 * P * L));
    for (int l = 0; l < L; ++l) std::memcpy(o->layers + 2 * 3 * P * l, r.layers[l].data.data(), sizeof(double) * 2 * 3 * P);
    o->t_final = static_cast<double*>(std::malloc(sizeof(double) * r.t_final.size()));
    std::memcpy(o->t_final, r.t_final.data(), sizeof(double) * r.t_final.size());
    o->n_contrib = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * r.n_contrib.size()));
    std::memcpy(o->n_contrib, r.n_contrib.data(), sizeof(int32_t) * r.n_contrib.size());
    o->projected = static_cast<ho_projected*>(std::calloc(N ? N : 1, sizeof(ho_projected)));
    for (size_t i = 0; i < N; ++i) {
        const auto& p = r.projected[i];
        ho_projected& q = o->projected[i];
        q.valid = p.valid;
        q.n = p.n;
        q.mu_x = p.mu_x;
        q.mu_y = p.mu_y;
        q.inv00 = p.inv00;
        q.inv01 = p.inv01;
        q.inv11 = p.inv11;
        q.radius = p.radius;
        q.xc = p.xc;
        q.yc = p.yc;
        q.zc = p.zc;
        q.alpha_sig = p.alpha_sig;
        for (int c = 0; c < 3; ++c) {
            q.amp[c] = p.amp[c];
            q.phase[c] = p.phase[c];
        }
        q.plane = p.plane;
    }
    o->rho = static_cast<double*>(std::malloc(sizeof(double) * (r.rho.size() + 1)));
    std::memcpy(o->rho, r.rho.data(), sizeof(double) * r.rho.size());
    o->touched = static_cast<uint8_t*>(std::malloc(N + 1));
    std::memcpy(o->touched, r.touched.data(), N);
    o->entry_bucket = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (E + 1)));
    o->entry_gidx = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (E + 1)));
    o->entry_depth = static_cast<double*>(std::malloc(sizeof(double) * (E + 1)));
    for (size_t e = 0; e < E; ++e) {
        o->entry_bucket[e] = r.entries[e].bucket;
        o->entry_gidx[e] = r.entries[e].gidx;
        o->entry_depth[e] = r.entries[e].depth;
    }
    o->bucket_start = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * r.bucket_start.size()));
    std::memcpy(o->bucket_start, r.bucket_start.data(), sizeof(uint32_t) * r.bucket_start.size());
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return HO_OK;
    } catch (const holo::HoloError& e) {
        g_err = e.what();
        return code_for(e);
    } catch (const std::exception& e) {
        g_err = e.what();
        return HO_ERR_NUMERIC;
    }
}

double secs(std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_raster_free(ho_raster* r) {
    if (!r) return;
    std::free(r->layers);
    std::free(r->t_final);
    std::free(r->n_contrib);
    std::free(r->projected);
    std::free(r->rho);
    std::free(r->touched);
    std::free(r->entry_bucket);
    std::free(r->entry_gidx);
    std::free(r->entry_depth);
    std::free(r->bucket_start);
    std::memset(r, 0, sizeof *r);
}

int ref_raster_forward(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                       ho_raster* out) {
    return guarded([&] {
        const holo::RasterForward r = holo::raster_forward(to_scene(s), to_camera(cam), to_wave(cfg), to_settings(st));
        copy_raster(r, cfg->num_planes, cfg->nx, cfg->ny, out);
    });
}

int ref_brute_force_forward(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                            double* layers) {
    return guarded([&] {
        const auto ls = holo::brute_force_forward(to_scene(s), to_camera(cam), to_wave(cfg), to_settings(st));
        const size_t n = ls.empty() ? 0 : ls[0].data.size();
        for (size_t l = 0; l < ls.size(); ++l) std::memcpy(layers + 2 * n * l, ls[l].data.data(), sizeof(double) * 2 * n);
    });
}

int ref_fft2(double* data, int w, int h, int inverse) {
    return guarded([&] {
        if (inverse)
            holo::ifft2(reinterpret_cast<holo::c64*>(data), w, h);
        else
            holo::fft2(reinterpret_cast<holo::c64*>(data), w, h);
    });
}

int ref_transfer_function(const ho_wave* cfg, double z, const ho_prop* opt, double* out) {
    return guarded([&] {
        const holo::TransferFunction tf = holo::transfer_function(to_wave(cfg), z, to_prop(opt));
        std::memcpy(out, tf.hz.data(), sizeof(double) * 2 * tf.hz.size());
    });
}

int ref_propagate(const double* in, int w, int h, int c, const ho_wave* cfg, double z, const ho_prop* opt,
                  double* out) {
    return guarded([&] {
        const holo::ComplexField r = holo::propagate(to_field(in, w, h, c, cfg->pitch), to_wave(cfg), z, to_prop(opt));
        std::memcpy(out, r.data.data(), sizeof(double) * 2 * r.data.size());
    });
}

int ref_forward_record(const double* layers, int L, int c, const ho_wave* cfg, const ho_prop* opt, double* holo_out) {
    return guarded([&] {
        std::vector<holo::ComplexField> ls;
        const size_t n = static_cast<size_t>(cfg->nx) * cfg->ny * c;
        for (int l = 0; l < L; ++l) ls.push_back(to_field(layers + 2 * n * l, cfg->nx, cfg->ny, c, cfg->pitch));
        const holo::ComplexField r = holo::forward_record(ls, to_wave(cfg), to_prop(opt));
        std::memcpy(holo_out, r.data.data(), sizeof(double) * 2 * r.data.size());
    });
}

int ref_inverse_propagate(const double* holo_in, int c, const ho_wave* cfg, const ho_prop* opt, double* replayed) {
    return guarded([&] {
        const auto rs = holo::inverse_propagate(to_field(holo_in, cfg->nx, cfg->ny, c, cfg->pitch), to_wave(cfg),
                                                to_prop(opt));
        const size_t n = rs.empty() ? 0 : rs[0].data.size();
        for (size_t l = 0; l < rs.size(); ++l) std::memcpy(replayed + 2 * n * l, rs[l].data.data(), sizeof(double) * 2 * n);
    });
}

// holo::pipeline_forward (pipeline.cpp:20-29), stage by stage so each stage is
// timed; for cfg->channels == 3 this is exactly the reference composition.  For
// fewer channels it is the SURVEY.md 8c adapter: the reference rasteriser always
// emits 3 channels, channels [0, C) are recorded and replayed.
int ref_pipeline_forward(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                         const ho_prop* opt, ho_raster* raster_out, double* hologram, double* replayed,
                         double* intensities, double* stage_seconds) {
    return guarded([&] {
        const holo::WaveConfig wc = to_wave(cfg);
        const holo::PropagationOptions po = to_prop(opt);
        const holo::GaussianScene scene = to_scene(s);
        const auto t0 = std::chrono::steady_clock::now();
        holo::RasterForward r = holo::raster_forward(scene, to_camera(cam), wc, to_settings(st));
        const auto t1 = std::chrono::steady_clock::now();
        std::vector<holo::ComplexField> layers;
        if (wc.channels() == holo::GaussianScene::kChannels) {
            layers = r.layers;
        } else {
            const size_t n = static_cast<size_t>(wc.nx) * wc.ny * wc.channels();
            for (const auto& f : r.layers) {
                holo::ComplexField g(wc.nx, wc.ny, wc.channels(), wc.pitch);
                std::memcpy(g.data.data(), f.data.data(), sizeof(double) * 2 * n);
                layers.push_back(std::move(g));
            }
        }
        const auto t1b = std::chrono::steady_clock::now();
        const holo::ComplexField holo_f = holo::forward_record(layers, wc, po);
        const auto t2 = std::chrono::steady_clock::now();
        const auto rep = holo::inverse_propagate(holo_f, wc, po);
        const auto t3 = std::chrono::steady_clock::now();
        std::vector<holo::IntensityImage> ints;
        ints.reserve(rep.size());
        for (const auto& v : rep) ints.push_back(holo::intensity(v));
        const auto t4 = std::chrono::steady_clock::now();
        const size_t n = holo_f.data.size();
        if (hologram) std::memcpy(hologram, holo_f.data.data(), sizeof(double) * 2 * n);
        for (size_t l = 0; l < rep.size(); ++l) {
            if (replayed) std::memcpy(replayed + 2 * n * l, rep[l].data.data(), sizeof(double) * 2 * n);
            if (intensities) std::memcpy(intensities + n * l, ints[l].data.data(), sizeof(double) * n);
        }
        if (raster_out) copy_raster(r, cfg->num_planes, cfg->nx, cfg->ny, raster_out);
        if (stage_seconds) {
            stage_seconds[0] = secs(t0, t1);
            stage_seconds[1] = secs(t1b, t2);
            stage_seconds[2] = secs(t2, t3);
            stage_seconds[3] = secs(t3, t4);
        }
    });
}

// Gradient outputs (caller-allocated, scene-shaped; mu_screen is N x 2).
struct ref_grads {
    double *positions, *rotations, *log_scales, *amplitudes, *opacity_logits, *phases, *plane_logits, *mu_screen;
};

static void copy_grads(const holo::SceneGradients& g, ref_grads* o) {
    auto put = [](const std::vector<double>& v, double* d) {
        if (d && !v.empty()) std::memcpy(d, v.data(), sizeof(double) * v.size());
    };
    put(g.positions, o->positions);
    put(g.rotations, o->rotations);
    put(g.log_scales, o->log_scales);
    put(g.amplitudes, o->amplitudes);
    put(g.opacity_logits, o->opacity_logits);
    put(g.phases, o->phases);
    put(g.plane_logits, o->plane_logits);
    put(g.mu_screen, o->mu_screen);
}

// holo::raster_backward (rasterizer.cpp:332-528) after holo::raster_forward;
// grad_layers: [L][3][H][W] complex128.
int ref_raster_backward(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                        const double* grad_layers, ref_grads* out) {
    return guarded([&] {
        const holo::GaussianScene scene = to_scene(s);
        const holo::WaveConfig wc = to_wave(cfg);
        const holo::RenderSettings rs = to_settings(st);
        const holo::RasterForward r = holo::raster_forward(scene, to_camera(cam), wc, rs);
        std::vector<holo::ComplexField> gl;
        const size_t n = static_cast<size_t>(cfg->nx) * cfg->ny * 3;
        for (int l = 0; l < cfg->num_planes; ++l) gl.push_back(to_field(grad_layers + 2 * n * l, cfg->nx, cfg->ny, 3, cfg->pitch));
        copy_grads(holo::raster_backward(scene, to_camera(cam), wc, rs, r, gl), out);
    });
}

// The gradient branch of holo::total_loss (pipeline.cpp:63-80) for a given
// dL/d(intensities) [L][C][H][W] (f64), C = 3: pipeline_forward, the adjoint of
// the replay and of the recording, then raster_backward.  grad_hologram [C][H][W]
// and grad_layers [L][C][H][W] (complex128) are optional outputs.  The loss terms
// themselves (losses.cpp) are not on this path.
int ref_pipeline_backward(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                          const ho_prop* opt, const double* grad_intensities, double* grad_hologram,
                          double* grad_layers, ref_grads* out) {
    return guarded([&] {
        const holo::GaussianScene scene = to_scene(s);
        const holo::WaveConfig wc = to_wave(cfg);
        holo::PipelineOptions po;
        po.raster = to_settings(st);
        po.prop = to_prop(opt);
        const holo::PipelineForward f = holo::pipeline_forward(scene, to_camera(cam), wc, po);
        const size_t P = static_cast<size_t>(wc.nx) * wc.ny * wc.channels();
        const auto z = holo::plane_positions(wc);
        holo::ComplexField gh(wc.nx, wc.ny, wc.channels(), wc.pitch);
        for (size_t l = 0; l < f.replayed.size(); ++l) {  // pipeline.cpp:66-73
            holo::ComplexField gv = f.replayed[l];
            for (size_t i = 0; i < gv.data.size(); ++i) gv.data[i] = 2.0 * gv.data[i] * grad_intensities[l * P + i];
            const holo::ComplexField gp = holo::propagate(gv, wc, z[l], po.prop);
            for (size_t i = 0; i < gp.data.size(); ++i) gh.data[i] += gp.data[i];
        }
        std::vector<holo::ComplexField> gl;  // pipeline.cpp:75-78
        for (size_t l = 0; l < z.size(); ++l) gl.push_back(holo::propagate(gh, wc, -z[l], po.prop));
        if (grad_hologram) std::memcpy(grad_hologram, gh.data.data(), sizeof(double) * 2 * P);
        for (size_t l = 0; l < gl.size(); ++l)
            if (grad_layers) std::memcpy(grad_layers + 2 * P * l, gl[l].data.data(), sizeof(double) * 2 * P);
        copy_grads(holo::raster_backward(scene, to_camera(cam), wc, po.raster, f.raster, gl), out);
    });
}

// The loss terms of total_loss (pipeline.cpp:43-45, losses.cpp) on given focal
// stacks I, I_gt ([L][C][H][W] f64) and masks ([L][H][W] f64, ignored when plain):
// out = {recon, ssim}; psnr [L]; grad [L][C][H][W] (dL/dI, written).
int ref_losses(const double* I, const double* I_gt, const double* masks, int L, int C, int H, int W,
               double lambda_ssim, int plain, double* out, double* psnr_out, double* grad) {
    return guarded([&] {
        const size_t n = static_cast<size_t>(C) * H * W, P = static_cast<size_t>(H) * W;
        std::vector<holo::IntensityImage> a, b, m, g;
        for (int l = 0; l < L; ++l) {
            a.emplace_back(W, H, C);
            b.emplace_back(W, H, C);
            m.emplace_back(W, H, 1);
            g.emplace_back(W, H, C);
            std::memcpy(a.back().data.data(), I + l * n, sizeof(double) * n);
            std::memcpy(b.back().data.data(), I_gt + l * n, sizeof(double) * n);
            if (masks) std::memcpy(m.back().data.data(), masks + l * P, sizeof(double) * P);
        }
        out[0] = plain ? holo::loss_mse(a, b, &g) : holo::loss_recon(a, b, m, &g);
        out[1] = holo::loss_ssim(a, b, lambda_ssim, &g);
        for (int l = 0; l < L; ++l) {
            if (psnr_out) psnr_out[l] = holo::psnr(a[l], b[l]);
            if (grad) std::memcpy(grad + l * n, g[l].data.data(), sizeof(double) * n);
        }
    });
}

// holo::total_loss (pipeline.cpp:30-95) with grads: breakdown = {recon, ssim,
// opacity, total, psnr_mean}; psnr [L]; targets [L][C][H][W], masks [L][H][W].
int ref_total_loss(const ho_scene* s, const ho_camera* cam, const ho_wave* cfg, const ho_settings* st,
                   const ho_prop* opt, double lambda_ssim, double lambda_opacity, int plain, const double* targets,
                   const double* masks, double* breakdown, double* psnr_out, ref_grads* grads) {
    return guarded([&] {
        const holo::GaussianScene scene = to_scene(s);
        const holo::WaveConfig wc = to_wave(cfg);
        holo::PipelineOptions po;
        po.raster = to_settings(st);
        po.prop = to_prop(opt);
        po.lambda_ssim = lambda_ssim;
        po.lambda_opacity = lambda_opacity;
        po.use_plain_mse = plain != 0;
        holo::FocalStackTarget t;
        t.camera = to_camera(cam);
        const size_t n = static_cast<size_t>(wc.nx) * wc.ny * wc.channels(), P = static_cast<size_t>(wc.nx) * wc.ny;
        for (int l = 0; l < wc.num_planes; ++l) {
            t.images.emplace_back(wc.nx, wc.ny, wc.channels());
            t.masks.emplace_back(wc.nx, wc.ny, 1);
            std::memcpy(t.images.back().data.data(), targets + l * n, sizeof(double) * n);
            std::memcpy(t.masks.back().data.data(), masks + l * P, sizeof(double) * P);
        }
        holo::SceneGradients g;
        const holo::LossBreakdown lb = holo::total_loss(scene, t.camera, wc, t, po, grads ? &g : nullptr);
        breakdown[0] = lb.recon;
        breakdown[1] = lb.ssim;
        breakdown[2] = lb.opacity;
        breakdown[3] = lb.total;
        breakdown[4] = lb.psnr_mean;
        for (size_t l = 0; l < lb.psnr.size(); ++l)
            if (psnr_out) psnr_out[l] = lb.psnr[l];
        if (grads) copy_grads(g, grads);
    });
}

// holo::optimizer_step (optimizer.cpp:102-133) applied `steps` times from fresh
// moments, step k using grads + k * grad_stride (each a scene-shaped ref_grads
// layout packed as positions | rotations | log_scales | amplitudes | opacity |
// phases | plane_logits).  The scene arrays are updated in place; applied[k]
// records whether step k was taken.
int ref_optimizer_run(ho_scene* s, const double* grads, int steps, const double* cfgv, int use_adam,
                      long long schedule_total, int* applied) {
    return guarded([&] {
        holo::GaussianScene scene = to_scene(s);
        holo::OptimizerConfig oc;
        oc.lr_positions = cfgv[0];
        oc.lr_rotations = cfgv[1];
        oc.lr_log_scales = cfgv[2];
        oc.lr_amplitudes = cfgv[3];
        oc.lr_phases = cfgv[4];
        oc.lr_opacities = cfgv[5];
        oc.lr_plane_logits = cfgv[6];
        oc.beta1 = cfgv[7];
        oc.beta2 = cfgv[8];
        oc.beta3 = cfgv[9];
        oc.eps = cfgv[10];
        oc.lr_floor = cfgv[11];
        oc.use_adam = use_adam != 0;
        oc.schedule_total = schedule_total;
        holo::OptimState st;
        st.resize_like(scene);
        const size_t n = scene.size(), L = static_cast<size_t>(scene.num_planes);
        const size_t stride = n * (3 + 4 + 3 + 3 + 1 + 3 + L);
        for (int k = 0; k < steps; ++k) {
            const double* p = grads + k * stride;
            holo::SceneGradients g;
            g.resize_like(scene);
            for (auto* v : {&g.positions, &g.rotations, &g.log_scales, &g.amplitudes, &g.opacity_logits, &g.phases,
                            &g.plane_logits}) {
                std::memcpy(v->data(), p, sizeof(double) * v->size());
                p += v->size();
            }
            applied[k] = holo::optimizer_step(st, scene, g, oc) ? 1 : 0;
        }
        std::memcpy(const_cast<double*>(s->positions), scene.positions.data(), sizeof(double) * 3 * n);
        std::memcpy(const_cast<double*>(s->rotations), scene.rotations.data(), sizeof(double) * 4 * n);
        std::memcpy(const_cast<double*>(s->log_scales), scene.log_scales.data(), sizeof(double) * 3 * n);
        std::memcpy(const_cast<double*>(s->amplitudes), scene.amplitudes.data(), sizeof(double) * 3 * n);
        std::memcpy(const_cast<double*>(s->opacity_logits), scene.opacity_logits.data(), sizeof(double) * n);
        std::memcpy(const_cast<double*>(s->phases), scene.phases.data(), sizeof(double) * 3 * n);
        std::memcpy(const_cast<double*>(s->plane_logits), scene.plane_logits.data(), sizeof(double) * n * L);
    });
}

}  // extern "C"

// ---- phase-only conversion (phase_only.cpp) on interleaved complex128 [C][H][W]
extern "C" {

int ref_phase_only_loss(const double* P, const double* theta, const ho_wave* cfg, double lambda_ssim,
                        const ho_prop* prop, int use_adam, double* loss, double* grad) {
    return guarded([&] {
        const holo::WaveConfig wc = to_wave(cfg);
        const holo::ComplexField f = to_field(P, wc.nx, wc.ny, wc.channels(), wc.pitch);
        holo::PhaseOnlyOptions opt;
        opt.lambda_ssim = lambda_ssim;
        opt.prop = to_prop(prop);
        opt.use_adam = use_adam != 0;
        std::vector<double> th(theta, theta + f.data.size()), g;
        *loss = holo::phase_only_loss(f, th, wc, opt, grad ? &g : nullptr);
        if (grad) std::memcpy(grad, g.data(), sizeof(double) * g.size());
    });
}

int ref_convert_phase_only(const double* P, const ho_wave* cfg, int iters, double lr, double lambda_ssim,
                           const ho_prop* prop, int use_adam, double* phase_out, double* trace) {
    return guarded([&] {
        const holo::WaveConfig wc = to_wave(cfg);
        const holo::ComplexField f = to_field(P, wc.nx, wc.ny, wc.channels(), wc.pitch);
        holo::PhaseOnlyOptions opt;
        opt.lambda_ssim = lambda_ssim;
        opt.prop = to_prop(prop);
        opt.use_adam = use_adam != 0;
        const holo::PhaseOnlyResult r = holo::convert_phase_only(f, wc, iters, lr, opt);
        std::memcpy(phase_out, r.hologram.phase.data(), sizeof(double) * r.hologram.phase.size());
        std::memcpy(trace, r.trace.data(), sizeof(double) * r.trace.size());
    });
}

}  // extern "C"
