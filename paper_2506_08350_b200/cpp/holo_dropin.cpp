// libholo.so — the reference's render-path C++ API (proj/include/holo/*.hpp)
// implemented over libholo_cuda's C-ABI (include/holo_cuda.h).
//
// Host-side pieces that are not compute (configuration, validation, camera
// rotation, scene bookkeeping, HOLOFIELD I/O, the energy / dot_real reductions
// the reference uses as test metrics, the analytic point-source field) are
// plain C++ here; every transform, propagation, rasterisation and the render
// itself run on the GPU.  There is no CPU fallback: without a CUDA device the
// calls throw HoloError("cuda", ...).
#include <cuda_runtime.h>

#include <algorithm>
#include <bit>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <thread>
#include <type_traits>
#include <omp.h>

#include "holo/camera.hpp"
#include "holo/device.hpp"
#include "holo/fft.hpp"
#include "holo/field.hpp"
#include "holo/field_io.hpp"
#include "holo/losses.hpp"
#include "holo/optimizer.hpp"
#include "holo/phase_only.hpp"
#include "holo/pipeline.hpp"
#include "holo/propagation.hpp"
#include "holo/rasterizer.hpp"
#include "holo/scene.hpp"
#include "holo/scene_io.hpp"
#include "holo/ssim.hpp"
#include "holo/wave_config.hpp"
#include "holo_cuda.h"

namespace holo {

// ------------------------------------------------------------------ device plumbing

namespace {

thread_local int t_device = 0;
thread_local bool t_f64 = true;

void check(int rc) {
    if (rc == HOLO_OK) return;
    static const char* kinds[] = {"", "config", "io", "usage", "numeric", "cuda", "oom", "nccl"};
    throw HoloError(rc > 0 && rc < 8 ? kinds[rc] : "numeric", holo_last_error());
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw HoloError("cuda", std::string(what) + ": " + cudaGetErrorString(e));
}

struct CtxHolder {
    holo_ctx* h = nullptr;
    ~CtxHolder() {
        if (h) holo_ctx_destroy(h);
    }
};

holo_ctx* ctx() {
    thread_local CtxHolder c;
    if (!c.h) check(holo_ctx_create(t_device, &c.h));
    return c.h;
}

cudaStream_t stream() { return static_cast<cudaStream_t>(holo_ctx_get_stream(ctx())); }

struct DevMem {
    void* p = nullptr;
    explicit DevMem(size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc"); }
    ~DevMem() { cudaFree(p); }
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
};

// The value-semantics API moves large host arrays in and out every call.  Large
// transfers go through a pinned staging pair per thread (pageable cudaMemcpy runs
// at a fraction of PCIe bandwidth), and the host-side copy between the staging
// buffer and the caller's memory -- including the first-touch page faults of a
// freshly allocated result -- runs on all cores, overlapped with the next chunk's
// DMA.
struct Staging {
    static constexpr size_t kChunk = size_t{32} << 20;
    unsigned char* buf[2] = {};
    cudaEvent_t ev[2] = {};
    Staging() {
        for (int k = 0; k < 2; ++k) {
            cuda_check(cudaMallocHost(reinterpret_cast<void**>(&buf[k]), kChunk), "cudaMallocHost");
            cuda_check(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming), "cudaEventCreate");
        }
    }
    ~Staging() {
        for (int k = 0; k < 2; ++k) {
            if (ev[k]) cudaEventSynchronize(ev[k]), cudaEventDestroy(ev[k]);
            if (buf[k]) cudaFreeHost(buf[k]);
        }
    }
};
Staging& staging() {
    thread_local Staging s;
    return s;
}
constexpr size_t kStagedMin = size_t{4} << 20;

void par_copy(void* dst, const void* src, size_t n) {
    constexpr size_t kBlk = size_t{1} << 20;
    const long nb = static_cast<long>((n + kBlk - 1) / kBlk);
#pragma omp parallel for schedule(static)
    for (long i = 0; i < nb; ++i) {
        const size_t o = static_cast<size_t>(i) * kBlk;
        std::memcpy(static_cast<unsigned char*>(dst) + o, static_cast<const unsigned char*>(src) + o,
                    std::min(kBlk, n - o));
    }
}

void h2d(void* d, const void* h, size_t n) {
    if (n < kStagedMin) {
        cuda_check(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, stream()), "cudaMemcpyAsync H2D");
        return;
    }
    Staging& st = staging();
    for (size_t off = 0, i = 0; off < n; off += Staging::kChunk, ++i) {
        const int k = static_cast<int>(i & 1);
        const size_t len = std::min(Staging::kChunk, n - off);
        cuda_check(cudaEventSynchronize(st.ev[k]), "cudaEventSynchronize");  // the buffer's last DMA is done
        par_copy(st.buf[k], static_cast<const unsigned char*>(h) + off, len);
        cuda_check(cudaMemcpyAsync(static_cast<unsigned char*>(d) + off, st.buf[k], len, cudaMemcpyHostToDevice,
                                   stream()),
                   "cudaMemcpyAsync H2D");
        cuda_check(cudaEventRecord(st.ev[k], stream()), "cudaEventRecord");
    }
}

void d2h(void* h, const void* d, size_t n) {
    if (n < kStagedMin) {
        cuda_check(cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, stream()), "cudaMemcpyAsync D2H");
        cuda_check(cudaStreamSynchronize(stream()), "cudaStreamSynchronize");
        return;
    }
    Staging& st = staging();
    auto issue = [&](size_t i) {
        const size_t off = i * Staging::kChunk;
        const int k = static_cast<int>(i & 1);
        cuda_check(cudaEventSynchronize(st.ev[k]), "cudaEventSynchronize");
        cuda_check(cudaMemcpyAsync(st.buf[k], static_cast<const unsigned char*>(d) + off,
                                   std::min(Staging::kChunk, n - off), cudaMemcpyDeviceToHost, stream()),
                   "cudaMemcpyAsync D2H");
        cuda_check(cudaEventRecord(st.ev[k], stream()), "cudaEventRecord");
    };
    const size_t chunks = (n + Staging::kChunk - 1) / Staging::kChunk;
    issue(0);
    for (size_t i = 0; i < chunks; ++i) {
        const int k = static_cast<int>(i & 1);
        cuda_check(cudaEventSynchronize(st.ev[k]), "cudaEventSynchronize");
        if (i + 1 < chunks) issue(i + 1);  // the other buffer's host copy finished last iteration
        const size_t off = i * Staging::kChunk;
        par_copy(static_cast<unsigned char*>(h) + off, st.buf[k], std::min(Staging::kChunk, n - off));
    }
}

// complex64 device samples -> complex<double> host samples, in staged chunks:
// double-buffered, the next chunk's DMA in flight while this one is widened
void d2h_widen(c64* h, const void* d, size_t n) {
    Staging& st = staging();
    constexpr size_t kPer = Staging::kChunk / sizeof(std::complex<float>);
    const size_t chunks = (n + kPer - 1) / kPer;
    auto issue = [&](size_t i) {
        const int k = static_cast<int>(i & 1);
        const size_t off = i * kPer;
        cuda_check(cudaEventSynchronize(st.ev[k]), "cudaEventSynchronize");
        cuda_check(cudaMemcpyAsync(st.buf[k], static_cast<const std::complex<float>*>(d) + off,
                                   std::min(kPer, n - off) * sizeof(std::complex<float>), cudaMemcpyDeviceToHost,
                                   stream()),
                   "cudaMemcpyAsync D2H");
        cuda_check(cudaEventRecord(st.ev[k], stream()), "cudaEventRecord");
    };
    if (chunks > 0) issue(0);
    for (size_t i = 0; i < chunks; ++i) {
        const int k = static_cast<int>(i & 1);
        cuda_check(cudaEventSynchronize(st.ev[k]), "cudaEventSynchronize");
        if (i + 1 < chunks) issue(i + 1);  // the other buffer was widened last iteration
        const size_t off = i * kPer, len = std::min(kPer, n - off);
        const auto* src = reinterpret_cast<const std::complex<float>*>(st.buf[k]);
#pragma omp parallel for schedule(static)
        for (long j = 0; j < static_cast<long>(len); ++j) h[off + j] = c64(src[j].real(), src[j].imag());
    }
}

// count fields (or images) of one shape, allocated and zero-filled by parallel
// threads: the first touch of fresh host pages is the cost of large results
template <class T>
std::vector<T> make_parallel(int count, int w, int h, int c, double pitch) {
    std::vector<T> out(static_cast<size_t>(count));
#pragma omp parallel for schedule(static, 1)
    for (int l = 0; l < count; ++l) {
        if constexpr (std::is_same_v<T, ComplexField>)
            out[l] = T(w, h, c, pitch);
        else
            out[l] = T(w, h, c);
    }
    return out;
}

holo_wave to_c(const WaveConfig& w) {
    holo_wave c{};
    c.nx = w.nx;
    c.ny = w.ny;
    c.pitch = w.pitch;
    if (w.channels() > HOLO_MAX_CHANNELS) throw HoloError("config", "too many wavelength channels");
    c.channels = w.channels();
    for (int i = 0; i < c.channels; ++i) c.wavelengths[i] = w.wavelengths[i];
    c.distance = w.distance;
    c.volume_depth = w.volume_depth;
    c.num_planes = w.num_planes;
    return c;
}

holo_camera to_c(const CameraView& v) {
    holo_camera c{};
    for (int i = 0; i < 6; ++i) c.pose[i] = v.pose[i];
    c.focal_px = v.focal_px;
    c.cx = v.cx;
    c.cy = v.cy;
    c.width = v.width;
    c.height = v.height;
    return c;
}

holo_raster_settings to_c(const RenderSettings& s) {
    return {s.near_clip, s.dilation,  s.plane_eps, s.term_eps, s.alpha_floor, s.alpha_clamp, s.radius_form_cap,
            s.ste_tau,   s.soft_assignment ? 1 : 0, s.soft_tau, s.tile};
}

holo_prop_options to_c(const PropagationOptions& o) { return {o.pad2x ? 1 : 0, o.local_band_limit ? 1 : 0}; }

int dtype() { return t_f64 ? HOLO_F64 : HOLO_F32; }

// Upload a host complex<double> array in the operator precision.
void upload_field(void* d, const c64* h, size_t n) {
    if (t_f64) {
        h2d(d, h, sizeof(c64) * n);
        return;
    }
    std::vector<std::complex<float>> tmp(n);
    for (size_t i = 0; i < n; ++i) tmp[i] = std::complex<float>(static_cast<float>(h[i].real()), static_cast<float>(h[i].imag()));
    h2d(d, tmp.data(), sizeof(std::complex<float>) * n);
    cuda_check(cudaStreamSynchronize(stream()), "cudaStreamSynchronize");
}

void download_field(c64* h, const void* d, size_t n) {
    if (t_f64) {
        d2h(h, d, sizeof(c64) * n);
        return;
    }
    std::vector<std::complex<float>> tmp(n);
    d2h(tmp.data(), d, sizeof(std::complex<float>) * n);
    for (size_t i = 0; i < n; ++i) h[i] = c64(tmp[i].real(), tmp[i].imag());
}

size_t elem() { return t_f64 ? sizeof(c64) : sizeof(std::complex<float>); }

}  // namespace

namespace device {
void set_device(int d) { t_device = d; }
void set_operator_precision(bool use_f64) { t_f64 = use_f64; }
bool operator_precision_f64() { return t_f64; }
}  // namespace device

// ------------------------------------------------------------------ wave_config (wave_config.cpp:5-30)

void WaveConfig::validate() const {
    if (nx <= 0 || ny <= 0) throw HoloError("config", "resolution must be positive");
    if (pitch <= 0.0) throw HoloError("config", "pixel pitch must be positive");
    if (wavelengths.empty()) throw HoloError("config", "at least one wavelength required");
    if (std::any_of(wavelengths.begin(), wavelengths.end(), [](double l) { return l <= 0.0; }))
        throw HoloError("config", "wavelengths must be positive");
    if (distance <= 0.0) throw HoloError("config", "propagation distance must be positive");
    if (volume_depth < 0.0) throw HoloError("config", "volume depth must be non-negative");
    if (num_planes < 1) throw HoloError("config", "need at least one depth plane");
    if (num_planes > 1 && volume_depth <= 0.0) throw HoloError("config", "multiple planes need a positive volume depth");
}

std::vector<double> plane_positions(const WaveConfig& cfg) {
    cfg.validate();
    const int L = cfg.num_planes;
    if (L == 1) return {cfg.distance};
    const double dz = cfg.volume_depth / (L - 1);
    const double z0 = cfg.distance - 0.5 * (L - 1) * dz;
    std::vector<double> z(L);
    for (int l = 0; l < L; ++l) z[l] = z0 + l * dz;
    return z;
}

// ------------------------------------------------------------------ field (field.cpp)

IntensityImage intensity(const ComplexField& u) {
    IntensityImage out(u.w, u.h, u.c);
    const size_t n = u.data.size();
    if (n == 0) return out;
    DevMem din(sizeof(c64) * n), dout(sizeof(double) * n);
    h2d(din.p, u.data.data(), sizeof(c64) * n);
    check(holo_intensity(ctx(), din.p, dout.p, n, HOLO_F64));
    d2h(out.data.data(), dout.p, sizeof(double) * n);
    return out;
}

double energy_channel(const ComplexField& u, int ch) {
    std::vector<double> rows(u.h, 0.0);
    const c64* base = u.channel(ch);
    for (int y = 0; y < u.h; ++y) {
        double s = 0.0;
        for (int x = 0; x < u.w; ++x) {
            const c64 v = base[static_cast<size_t>(y) * u.w + x];
            s += v.real() * v.real() + v.imag() * v.imag();
        }
        rows[y] = s;
    }
    return fold_partials(rows);
}

double energy(const ComplexField& u) {
    double s = 0.0;
    for (int ch = 0; ch < u.c; ++ch) s += energy_channel(u, ch);
    return s;
}

double dot_real(const ComplexField& a, const ComplexField& b) {
    if (!a.same_shape(b)) throw HoloError("numeric", "dot_real: shape mismatch");
    std::vector<double> rows(static_cast<size_t>(a.h) * a.c, 0.0);
    for (int ch = 0; ch < a.c; ++ch)
        for (int y = 0; y < a.h; ++y) {
            double s = 0.0;
            const c64* ra = a.channel(ch) + static_cast<size_t>(y) * a.w;
            const c64* rb = b.channel(ch) + static_cast<size_t>(y) * a.w;
            for (int x = 0; x < a.w; ++x) s += ra[x].real() * rb[x].real() + ra[x].imag() * rb[x].imag();
            rows[static_cast<size_t>(ch) * a.h + y] = s;
        }
    return fold_partials(rows);
}

// ------------------------------------------------------------------ fft (fft.cpp:33-44)

static void fft2_dir(c64* data, int w, int h, int inverse) {
    if (w <= 0 || h <= 0) throw HoloError("numeric", "fft2: dimensions must be positive");
    const size_t n = static_cast<size_t>(w) * h;
    DevMem d(sizeof(c64) * n);
    h2d(d.p, data, sizeof(c64) * n);
    check(holo_fft2(ctx(), d.p, w, h, 1, inverse, HOLO_F64));
    d2h(data, d.p, sizeof(c64) * n);
}

void fft2(c64* data, int w, int h) { fft2_dir(data, w, h, 0); }
void ifft2(c64* data, int w, int h) { fft2_dir(data, w, h, 1); }

// ------------------------------------------------------------------ propagation (propagation.cpp:86-167)

TransferFunction transfer_function(const WaveConfig& cfg, double z, const PropagationOptions& opt) {
    cfg.validate();
    TransferFunction tf;
    tf.w = opt.pad2x ? 2 * cfg.nx : cfg.nx;
    tf.h = opt.pad2x ? 2 * cfg.ny : cfg.ny;
    tf.c = cfg.channels();
    tf.z = z;
    tf.hz.resize(static_cast<size_t>(tf.w) * tf.h * tf.c);
    DevMem d(sizeof(c64) * tf.hz.size());
    const holo_wave w = to_c(cfg);
    const holo_prop_options po = to_c(opt);
    check(holo_transfer_function(ctx(), &w, z, &po, d.p, HOLO_F64));
    d2h(tf.hz.data(), d.p, sizeof(c64) * tf.hz.size());
    return tf;
}

ComplexField propagate(const ComplexField& u, const WaveConfig& cfg, double z, const PropagationOptions& opt) {
    if (u.w != cfg.nx || u.h != cfg.ny || u.c != cfg.channels())
        throw HoloError("config", "propagate: field does not match the configured grid");
    ComplexField out(u.w, u.h, u.c, u.pitch);
    const size_t n = u.data.size();
    DevMem din(elem() * n), dout(elem() * n);
    upload_field(din.p, u.data.data(), n);
    const holo_wave w = to_c(cfg);
    const holo_prop_options po = to_c(opt);
    check(holo_propagate(ctx(), din.p, dout.p, u.w, u.h, u.c, &w, z, &po, dtype()));
    download_field(out.data.data(), dout.p, n);
    return out;
}

ComplexField forward_record(const std::vector<ComplexField>& layers, const WaveConfig& cfg,
                            const PropagationOptions& opt) {
    const std::vector<double> zs = plane_positions(cfg);
    if (layers.size() != zs.size())
        throw HoloError("config", "forward_record: layer count does not match num_planes");
    for (const ComplexField& l : layers)
        if (l.w != cfg.nx || l.h != cfg.ny || l.c != cfg.channels())
            throw HoloError("config", "propagate: field does not match the configured grid");
    const size_t n = static_cast<size_t>(cfg.nx) * cfg.ny * cfg.channels();
    DevMem dl(elem() * n * layers.size()), dh(elem() * n);
    for (size_t l = 0; l < layers.size(); ++l)
        upload_field(static_cast<char*>(dl.p) + elem() * n * l, layers[l].data.data(), n);
    const holo_wave w = to_c(cfg);
    const holo_prop_options po = to_c(opt);
    check(holo_forward_record(ctx(), dl.p, static_cast<int>(layers.size()), dh.p, &w, &po, dtype()));
    ComplexField out(cfg.nx, cfg.ny, cfg.channels(), cfg.pitch);
    download_field(out.data.data(), dh.p, n);
    return out;
}

std::vector<ComplexField> inverse_propagate(const ComplexField& hologram, const WaveConfig& cfg,
                                            const PropagationOptions& opt) {
    const std::vector<double> zs = plane_positions(cfg);
    if (hologram.w != cfg.nx || hologram.h != cfg.ny || hologram.c != cfg.channels())
        throw HoloError("config", "propagate: field does not match the configured grid");
    const size_t n = hologram.data.size();
    DevMem dh(elem() * n), dr(elem() * n * zs.size());
    upload_field(dh.p, hologram.data.data(), n);
    const holo_wave w = to_c(cfg);
    const holo_prop_options po = to_c(opt);
    check(holo_inverse_propagate(ctx(), dh.p, dr.p, &w, &po, dtype()));
    std::vector<ComplexField> out;
    out.reserve(zs.size());
    for (size_t l = 0; l < zs.size(); ++l) {
        ComplexField f(cfg.nx, cfg.ny, cfg.channels(), cfg.pitch);
        download_field(f.data.data(), static_cast<const char*>(dr.p) + elem() * n * l, n);
        out.push_back(std::move(f));
    }
    return out;
}

double point_phase_exact(double lambda, double dx, double dy, double z) {
    return wrap_phase(kTwoPi * std::sqrt(dx * dx + dy * dy + z * z) / lambda);
}

double point_phase_paraxial(double lambda, double dx, double dy, double z) {
    return wrap_phase(kTwoPi * (z + (dx * dx + dy * dy) / (2.0 * z)) / lambda);
}

// Analytic spherical-wave field on the hologram grid (propagation.cpp:135-167); a
// validation oracle in the reference, evaluated directly here.
ComplexField point_source_field(const WaveConfig& cfg, const std::vector<PointSource>& sources,
                                const PointSourceOptions& opt) {
    cfg.validate();
    for (const PointSource& s : sources) {
        if (s.z <= 0.0) throw HoloError("config", "point sources must sit in front of the hologram plane");
        if (s.amps.size() != 1 && s.amps.size() != static_cast<size_t>(cfg.channels()))
            throw HoloError("config", "point source amplitude count must be 1 or match the channels");
    }
    const double ox = opt.cx >= 0.0 ? opt.cx : cfg.nx / 2.0;
    const double oy = opt.cy >= 0.0 ? opt.cy : cfg.ny / 2.0;
    ComplexField out(cfg.nx, cfg.ny, cfg.channels(), cfg.pitch);
    for (int ch = 0; ch < cfg.channels(); ++ch) {
        const double lambda = cfg.wavelengths[ch];
        for (const PointSource& s : sources) {
            const double amp = s.amps.size() == 1 ? s.amps[0] : s.amps[ch];
            for (int y = 0; y < cfg.ny; ++y) {
                const double py = ((y + 0.5) - oy) * cfg.pitch - s.y;
                for (int x = 0; x < cfg.nx; ++x) {
                    const double px = ((x + 0.5) - ox) * cfg.pitch - s.x;
                    const double phi = s.phase0 + (opt.paraxial ? point_phase_paraxial(lambda, px, py, s.z)
                                                                : point_phase_exact(lambda, px, py, s.z));
                    const double a = opt.inverse_r ? amp / std::sqrt(px * px + py * py + s.z * s.z) : amp;
                    out.at(ch, y, x) += c64(a * std::cos(phi), a * std::sin(phi));
                }
            }
        }
    }
    return out;
}

// ------------------------------------------------------------------ camera (camera.cpp)

Eigen::Matrix3d CameraView::rot_cam_to_world() const {
    const double ca = std::cos(pose[3]), sa = std::sin(pose[3]);
    const double cb = std::cos(pose[4]), sb = std::sin(pose[4]);
    const double cg = std::cos(pose[5]), sg = std::sin(pose[5]);
    Eigen::Matrix3d rx, ry, rz;
    rx << 1, 0, 0, 0, ca, -sa, 0, sa, ca;
    ry << cb, 0, sb, 0, 1, 0, -sb, 0, cb;
    rz << cg, -sg, 0, sg, cg, 0, 0, 0, 1;
    return rz * ry * rx;
}

Eigen::Matrix3d CameraView::rot_world_to_cam() const { return rot_cam_to_world().transpose(); }

Eigen::Vector3d CameraView::world_to_camera(const Eigen::Vector3d& p) const {
    return rot_world_to_cam() * (p - position());
}

void CameraView::validate() const {
    if (width <= 0 || height <= 0) throw HoloError("config", "camera resolution must be positive");
    if (focal_px <= 0.0) throw HoloError("config", "focal length must be positive");
    for (double v : pose)
        if (!std::isfinite(v)) throw HoloError("config", "camera pose must be finite");
}

// ------------------------------------------------------------------ scene (scene.cpp)

void GaussianScene::resize(size_t n) {
    positions.assign(n * 3, 0.0);
    rotations.assign(n * 4, 0.0);
    for (size_t i = 0; i < n; ++i) rotations[i * 4] = 1.0;
    log_scales.assign(n * 3, 0.0);
    amplitudes.assign(n * 3, 0.0);
    opacity_logits.assign(n, 0.0);
    phases.assign(n * 3, 0.0);
    plane_logits.assign(n * static_cast<size_t>(num_planes), 0.0);
}

static double quat_norm(const double* q) { return std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]); }

void GaussianScene::validate() const {
    const size_t n = size();
    if (num_planes < 1) throw HoloError("config", "scene needs at least one plane");
    if (positions.size() != n * 3 || rotations.size() != n * 4 || log_scales.size() != n * 3 ||
        amplitudes.size() != n * 3 || phases.size() != n * 3 || plane_logits.size() != n * static_cast<size_t>(num_planes))
        throw HoloError("config", "scene arrays have inconsistent sizes");
    for (size_t i = 0; i < n; ++i)
        if (!(quat_norm(&rotations[i * 4]) > 1e-8)) throw HoloError("config", "degenerate quaternion in scene");
    for (double a : amplitudes)
        if (a < 0.0) throw HoloError("config", "amplitudes must be non-negative");
}

void GaussianScene::renormalize() {
    for (size_t i = 0; i < size(); ++i) {
        double* q = &rotations[i * 4];
        const double nq = quat_norm(q);
        if (nq > 1e-12) {
            for (int k = 0; k < 4; ++k) q[k] /= nq;
        } else {
            q[0] = 1.0;
            q[1] = q[2] = q[3] = 0.0;
        }
    }
    for (double& a : amplitudes) a = std::max(a, 0.0);
}

namespace detail {
Eigen::Matrix3d quat_to_rot(const double* q) {
    const double n = quat_norm(q);
    const double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    Eigen::Matrix3d r;
    r << 1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y);
    return r;
}
}  // namespace detail

Eigen::Matrix3d covariance_3d(const double* quat, const double* log_scales) {
    const Eigen::Matrix3d R = detail::quat_to_rot(quat);
    Eigen::Matrix3d M = R;
    for (int k = 0; k < 3; ++k) {
        const double e = std::exp(log_scales[k]);
        for (int r = 0; r < 3; ++r) M(r, k) = R(r, k) * e;
    }
    return M * M.transpose();
}

SteAssign ste_assign(const double* logits, int L, double tau) {
    if (L < 1) throw HoloError("config", "ste_assign needs at least one plane");
    if (tau <= 0.0) throw HoloError("config", "ste temperature must be positive");
    SteAssign a;
    a.onehot.assign(L, 0.0);
    a.backward_weights.assign(L, 0.0);
    for (int l = 1; l < L; ++l)
        if (logits[l] > logits[a.index]) a.index = l;
    a.onehot[a.index] = 1.0;
    double denom = 0.0;
    for (int l = 0; l < L; ++l) denom += (a.backward_weights[l] = std::exp((logits[l] - logits[a.index]) / tau));
    for (double& v : a.backward_weights) v /= denom;
    return a;
}

// ------------------------------------------------------------------ rasterizer + pipeline (GPU)

namespace {

holo_scene_arrays scene_arrays(const GaussianScene& s) {
    return {s.size(),          s.num_planes,          s.positions.data(), s.rotations.data(),
            s.log_scales.data(), s.amplitudes.data(), s.opacity_logits.data(), s.phases.data(),
            s.plane_logits.data()};
}

// Upload a scene through a persistent pinned copy (the context's copy-in stream
// then runs at full PCIe bandwidth, asynchronously); the copy is reused once the
// previous upload from it has completed.
void upload_scene(const GaussianScene& s) {
    struct Pinned {
        double* p = nullptr;
        size_t cap = 0;
        ~Pinned() {
            if (p) cudaFreeHost(p);
        }
    };
    thread_local Pinned pin;
    const std::vector<double>* arr[7] = {&s.positions, &s.rotations, &s.log_scales, &s.amplitudes,
                                         &s.opacity_logits, &s.phases, &s.plane_logits};
    size_t total = 0;
    for (auto* a : arr) total += a->size();
    if (total * sizeof(double) < kStagedMin) {
        const holo_scene_arrays sa = scene_arrays(s);
        check(holo_scene_upload(ctx(), &sa));
        return;
    }
    cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(holo_ctx_get_copy_stream(ctx(), 0))),
               "cudaStreamSynchronize");  // the last upload from the pinned copy is done
    if (pin.cap < total) {
        if (pin.p) cudaFreeHost(pin.p);
        pin.p = nullptr;
        cuda_check(cudaMallocHost(reinterpret_cast<void**>(&pin.p), total * sizeof(double)), "cudaMallocHost");
        pin.cap = total;
    }
    const double* at[7];
    size_t o = 0;
    for (int k = 0; k < 7; ++k) {
        par_copy(pin.p + o, arr[k]->data(), arr[k]->size() * sizeof(double));
        at[k] = pin.p + o;
        o += arr[k]->size();
    }
    const holo_scene_arrays sa{s.size(), s.num_planes, at[0], at[1], at[2], at[3], at[4], at[5], at[6]};
    check(holo_scene_upload(ctx(), &sa));
}

void check_raster_inputs(const GaussianScene& scene, const CameraView& cam, const WaveConfig& cfg) {
    scene.validate();
    cam.validate();
    cfg.validate();
    if (scene.num_planes != cfg.num_planes) throw HoloError("config", "scene plane count does not match the wave config");
    if (cam.width != cfg.nx || cam.height != cfg.ny)
        throw HoloError("config", "camera resolution must match the hologram grid");
}

template <class T>
std::vector<T> download_buf(int which) {
    void* d = nullptr;
    size_t bytes = 0;
    check(holo_frame_buffer(ctx(), which, &d, &bytes));
    std::vector<T> h(bytes / sizeof(T));
    if (bytes) d2h(h.data(), d, bytes);
    return h;
}

// A frame buffer read whole into pinned host memory that is reused across calls
// (grown on demand): the source of element-wise conversions into the result
// arrays, without a zero-filled temporary vector and a second copy.
template <class T>
const T* download_pinned(int which, size_t& count, int slot) {
    struct Pinned {
        void* p = nullptr;
        size_t cap = 0;
        ~Pinned() {
            if (p) cudaFreeHost(p);
        }
    };
    thread_local Pinned pins[4];
    Pinned& pin = pins[slot];
    void* d = nullptr;
    size_t bytes = 0;
    check(holo_frame_buffer(ctx(), which, &d, &bytes));
    if (bytes > pin.cap) {
        if (pin.p) cudaFreeHost(pin.p);
        pin.p = nullptr;
        pin.cap = 0;
        cuda_check(cudaMallocHost(&pin.p, bytes), "cudaMallocHost");
        pin.cap = bytes;
    }
    if (bytes) {
        cuda_check(cudaMemcpyAsync(pin.p, d, bytes, cudaMemcpyDeviceToHost, stream()), "cudaMemcpyAsync D2H");
        cuda_check(cudaStreamSynchronize(stream()), "cudaStreamSynchronize");
    }
    count = bytes / sizeof(T);
    return static_cast<const T*>(pin.p);
}

detail::Projected to_projected(const holo_projected& q) {
    detail::Projected p;
    p.valid = q.valid != 0;
    p.n = q.n;
    p.mu_x = q.mu_x;
    p.mu_y = q.mu_y;
    p.inv00 = q.inv00;
    p.inv01 = q.inv01;
    p.inv11 = q.inv11;
    p.radius = q.radius;
    p.xc = q.xc;
    p.yc = q.yc;
    p.zc = q.zc;
    p.alpha_sig = q.alpha_sig;
    for (int c = 0; c < 3; ++c) {
        p.amp[c] = q.amp[c];
        p.phase[c] = q.phase[c];
    }
    p.plane = q.plane;
    return p;
}

std::vector<ComplexField> download_layers(const WaveConfig& cfg, int C) {
    const int L = cfg.num_planes, W = cfg.nx, H = cfg.ny;
    const size_t P = static_cast<size_t>(W) * H;
    void* d = nullptr;
    size_t bytes = 0;
    check(holo_frame_buffer(ctx(), HOLO_BUF_LAYERS, &d, &bytes));
    std::vector<ComplexField> out = make_parallel<ComplexField>(L, W, H, GaussianScene::kChannels, cfg.pitch);
    for (int l = 0; l < L; ++l)
        d2h_widen(out[l].data.data(), static_cast<const std::complex<float>*>(d) + static_cast<size_t>(l) * C * P,
                  static_cast<size_t>(C) * P);
    return out;
}

RasterForward collect_raster(const GaussianScene& scene, const WaveConfig& cfg, int C, const holo_frame_info& info) {
    RasterForward r;
    const int L = cfg.num_planes, W = cfg.nx, H = cfg.ny;
    const size_t P = static_cast<size_t>(W) * H, N = scene.size();
    r.tiles_x = info.tiles_x;
    r.tiles_y = info.tiles_y;
    const size_t B = static_cast<size_t>(L) * info.tiles_x * info.tiles_y;
    const size_t E = info.num_entries;
    // the result arrays are zero-filled by their constructors: side threads size
    // them while the main thread fills the layers (first touch of fresh pages is
    // the cost here)
    std::thread sizer1([&] {
        r.t_final.resize(L * P);
        r.projected.resize(N);
    });
    std::thread sizer2([&] {
        r.entries.resize(E);
        r.n_contrib.resize(L * P);
        r.rho.resize(N * L);
        r.touched.resize(N);
        r.bucket_start.resize(B + 1);
    });
    r.layers = download_layers(cfg, C);
    sizer1.join();
    sizer2.join();
    auto into = [&](int which, void* dst, size_t max_bytes) {
        void* d = nullptr;
        size_t bytes = 0;
        check(holo_frame_buffer(ctx(), which, &d, &bytes));
        if (bytes) d2h(dst, d, std::min(bytes, max_bytes));
    };
    size_t cnt = 0;
    const float* tf = download_pinned<float>(HOLO_BUF_T_FINAL, cnt, 0);
#pragma omp parallel for schedule(static)
    for (long i = 0; i < static_cast<long>(std::min(cnt, L * P)); ++i) r.t_final[i] = tf[i];
    into(HOLO_BUF_N_CONTRIB, r.n_contrib.data(), sizeof(std::int32_t) * L * P);
    const holo_projected* proj = download_pinned<holo_projected>(HOLO_BUF_PROJECTED, cnt, 1);
#pragma omp parallel for schedule(static)
    for (long i = 0; i < static_cast<long>(std::min(cnt, N)); ++i) r.projected[i] = to_projected(proj[i]);
    into(HOLO_BUF_RHO, r.rho.data(), sizeof(double) * N * L);
    into(HOLO_BUF_TOUCHED, r.touched.data(), N);
    into(HOLO_BUF_BUCKET_START, r.bucket_start.data(), sizeof(std::uint32_t) * (B + 1));
    size_t ng = 0, nd = 0;
    const std::int32_t* gidx = download_pinned<std::int32_t>(HOLO_BUF_ENTRY_GIDX, ng, 2);
    const double* depth = download_pinned<double>(HOLO_BUF_ENTRY_DEPTH, nd, 3);
    if (ng < E || nd < E) throw HoloError("numeric", "raster_forward: entry buffers shorter than the entry count");
#pragma omp parallel for schedule(dynamic, 256)
    for (long b = 0; b < static_cast<long>(B); ++b)
        for (std::uint32_t e = r.bucket_start[b]; e < r.bucket_start[b + 1]; ++e)
            r.entries[e] = detail::Entry{static_cast<std::int32_t>(b), gidx[e], depth[e]};
    return r;
}

constexpr unsigned kRasterOutputs = HOLO_OUT_LAYERS | HOLO_OUT_AUX | HOLO_OUT_LISTS | HOLO_OUT_PROJECTED;

}  // namespace

// rasterizer.cpp:139-263: always 3 channels of layers, like the reference
RasterForward raster_forward(const GaussianScene& scene, const CameraView& cam, const WaveConfig& cfg,
                             const RenderSettings& settings) {
    check_raster_inputs(scene, cam, cfg);
    upload_scene(scene);
    holo_wave w = to_c(cfg);
    w.channels = GaussianScene::kChannels;  // the rasteriser ignores wavelengths; it emits every scene channel
    for (int c = cfg.channels(); c < w.channels; ++c) w.wavelengths[c] = cfg.wavelengths.back();
    const holo_camera c = to_c(cam);
    const holo_raster_settings st = to_c(settings);
    const holo_prop_options po{0, 0};
    holo_frame_info info{};
    check(holo_render(ctx(), &c, &w, &st, &po, kRasterOutputs, &info));
    return collect_raster(scene, cfg, GaussianScene::kChannels, info);
}

// rasterizer.cpp:265-315 on the GPU (holo_brute_force_forward): same per-pixel math,
// global depth order, no tiles, no radius culling, no early termination
std::vector<ComplexField> brute_force_forward(const GaussianScene& scene, const CameraView& cam, const WaveConfig& cfg,
                                              const RenderSettings& settings) {
    check_raster_inputs(scene, cam, cfg);
    const holo_scene_arrays sa = scene_arrays(scene);
    check(holo_scene_upload(ctx(), &sa));
    holo_wave w = to_c(cfg);
    w.channels = GaussianScene::kChannels;
    for (int c = cfg.channels(); c < w.channels; ++c) w.wavelengths[c] = cfg.wavelengths.back();
    const holo_camera c = to_c(cam);
    const holo_raster_settings st = to_c(settings);
    check(holo_brute_force_forward(ctx(), &c, &w, &st));
    return download_layers(cfg, GaussianScene::kChannels);
}

namespace detail {
// rasterizer.cpp:10-70 for Gaussian n: the device projection of a one-Gaussian
// frame (f64, the same kernel as raster_forward's).  The device forms the
// rotation from the camera, so world_to_cam must be cam.rot_world_to_cam().
Projected project_gaussian(const GaussianScene& scene, size_t n, const CameraView& cam,
                           const Eigen::Matrix3d& world_to_cam, const WaveConfig& cfg, const RenderSettings& settings) {
    if (n >= scene.size()) throw HoloError("usage", "project_gaussian: index out of range");
    const Eigen::Matrix3d r = cam.rot_world_to_cam();
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            if (r(i, j) != world_to_cam(i, j))
                throw HoloError("usage", "project_gaussian: world_to_cam must be cam.rot_world_to_cam()");
    GaussianScene one;
    one.num_planes = scene.num_planes;
    one.resize(1);
    auto take = [n](const std::vector<double>& from, std::vector<double>& to, size_t k) {
        std::copy(from.begin() + static_cast<long>(n * k), from.begin() + static_cast<long>((n + 1) * k), to.begin());
    };
    take(scene.positions, one.positions, 3);
    take(scene.rotations, one.rotations, 4);
    take(scene.log_scales, one.log_scales, 3);
    take(scene.amplitudes, one.amplitudes, 3);
    take(scene.opacity_logits, one.opacity_logits, 1);
    take(scene.phases, one.phases, 3);
    take(scene.plane_logits, one.plane_logits, static_cast<size_t>(scene.num_planes));
    CameraView c = cam;
    c.width = cfg.nx;
    c.height = cfg.ny;
    const holo_scene_arrays sa = scene_arrays(one);
    check(holo_scene_upload(ctx(), &sa));
    holo_wave w = to_c(cfg);
    w.channels = GaussianScene::kChannels;
    for (int k = cfg.channels(); k < w.channels; ++k) w.wavelengths[k] = cfg.wavelengths.back();
    const holo_camera hc = to_c(c);
    const holo_raster_settings st = to_c(settings);
    const holo_prop_options po{0, 0};
    holo_frame_info info{};
    check(holo_render(ctx(), &hc, &w, &st, &po, HOLO_OUT_PROJECTED, &info));
    Projected p = to_projected(download_buf<holo_projected>(HOLO_BUF_PROJECTED).at(0));
    p.n = static_cast<int>(n);
    return p;
}
}  // namespace detail

void SceneGradients::resize_like(const GaussianScene& s) {
    const size_t n = s.size();
    positions.assign(3 * n, 0.0);
    rotations.assign(4 * n, 0.0);
    log_scales.assign(3 * n, 0.0);
    amplitudes.assign(3 * n, 0.0);
    opacity_logits.assign(n, 0.0);
    phases.assign(3 * n, 0.0);
    plane_logits.assign(n * static_cast<size_t>(s.num_planes), 0.0);
    mu_screen.assign(2 * n, 0.0);
}

void SceneGradients::clear() {
    for (auto* v : {&positions, &rotations, &log_scales, &amplitudes, &opacity_logits, &phases, &plane_logits,
                    &mu_screen})
        std::fill(v->begin(), v->end(), 0.0);
}

// rasterizer.cpp:332-528 on the device
SceneGradients raster_backward(const GaussianScene& scene, const CameraView& cam, const WaveConfig& cfg,
                               const RenderSettings& settings, const RasterForward& fwd,
                               const std::vector<ComplexField>& grad_layers) {
    const int L = cfg.num_planes;
    if (grad_layers.size() != static_cast<size_t>(L))
        throw HoloError("config", "raster_backward: upstream gradient count mismatch");  // rasterizer.cpp:342-343
    check_raster_inputs(scene, cam, cfg);
    if (fwd.projected.size() != scene.size()) throw HoloError("usage", "raster_backward: forward is for another scene");
    // the device keeps its own forward state: render the same frame there
    const holo_scene_arrays sa = scene_arrays(scene);
    check(holo_scene_upload(ctx(), &sa));
    holo_wave w = to_c(cfg);
    w.channels = GaussianScene::kChannels;
    for (int c = cfg.channels(); c < w.channels; ++c) w.wavelengths[c] = cfg.wavelengths.back();
    const holo_camera c = to_c(cam);
    const holo_raster_settings st = to_c(settings);
    const holo_prop_options po{0, 0};
    holo_frame_info info{};
    check(holo_render(ctx(), &c, &w, &st, &po, HOLO_OUT_LAYERS | HOLO_OUT_AUX, &info));
    const size_t P = static_cast<size_t>(cfg.nx) * cfg.ny, per = 3 * P;
    std::vector<std::complex<float>> g(static_cast<size_t>(L) * per);
    for (int l = 0; l < L; ++l) {
        if (grad_layers[l].c != 3 || grad_layers[l].w != cfg.nx || grad_layers[l].h != cfg.ny)
            throw HoloError("config", "raster_backward: upstream gradient shape mismatch");
        for (size_t i = 0; i < per; ++i)
            g[l * per + i] = std::complex<float>(static_cast<float>(grad_layers[l].data[i].real()),
                                                 static_cast<float>(grad_layers[l].data[i].imag()));
    }
    DevMem dg(sizeof(std::complex<float>) * g.size());
    h2d(dg.p, g.data(), sizeof(std::complex<float>) * g.size());
    SceneGradients out;
    out.resize_like(scene);
    std::vector<std::vector<double>*> vs = {&out.positions, &out.rotations, &out.log_scales, &out.amplitudes,
                                            &out.opacity_logits, &out.phases, &out.plane_logits, &out.mu_screen};
    std::vector<std::unique_ptr<DevMem>> dm;
    for (auto* v : vs) dm.push_back(std::make_unique<DevMem>(sizeof(double) * v->size()));
    holo_scene_grads hg{};
    double** slots[8] = {&hg.positions, &hg.rotations, &hg.log_scales, &hg.amplitudes,
                         &hg.opacity_logits, &hg.phases, &hg.plane_logits, &hg.mu_screen};
    for (int k = 0; k < 8; ++k) *slots[k] = static_cast<double*>(dm[k]->p);
    check(holo_raster_backward(ctx(), &c, &w, &st, dg.p, &hg));
    for (int k = 0; k < 8; ++k) d2h(vs[k]->data(), dm[k]->p, sizeof(double) * vs[k]->size());
    return out;
}

// pipeline.cpp:20-29
PipelineForward pipeline_forward(const GaussianScene& scene, const CameraView& cam, const WaveConfig& cfg,
                                 const PipelineOptions& opt) {
    check_raster_inputs(scene, cam, cfg);
    if (cfg.channels() != GaussianScene::kChannels)  // propagate's channel check (propagation.cpp:94-95)
        throw HoloError("config", "propagate: field does not match the configured grid");
    // HOLO_DROPIN_PROFILE=1: phase times of this call on stderr (measurement aid)
    static const bool prof = [] {
        const char* e = std::getenv("HOLO_DROPIN_PROFILE");
        return e && e[0] == '1';
    }();
    using clk = std::chrono::steady_clock;
    auto t_last = clk::now();
    auto lap = [&](const char* what) {
        if (!prof) return;
        const auto t = clk::now();
        std::fprintf(stderr, "pipeline_forward %s %.1f ms\n", what,
                     std::chrono::duration<double, std::milli>(t - t_last).count());
        t_last = t;
    };
    upload_scene(scene);
    lap("upload_scene");
    const holo_wave w = to_c(cfg);
    const holo_camera c = to_c(cam);
    const holo_raster_settings st = to_c(opt.raster);
    const holo_prop_options po = to_c(opt.prop);
    holo_frame_info info{};
    check(holo_render(ctx(), &c, &w, &st, &po,
                      kRasterOutputs | HOLO_OUT_HOLOGRAM | HOLO_OUT_REPLAYED | HOLO_OUT_INTENSITY, &info));
    lap("render");
    PipelineForward f;
    const int L = cfg.num_planes, C = cfg.channels();
    const size_t n = static_cast<size_t>(cfg.nx) * cfg.ny * C;
    f.raster = collect_raster(scene, cfg, C, info);
    lap("collect_raster");
    void* dholo = nullptr;
    void* drep0 = nullptr;
    size_t bytes0 = 0;
    check(holo_frame_buffer(ctx(), HOLO_BUF_HOLOGRAM, &dholo, &bytes0));
    check(holo_frame_buffer(ctx(), HOLO_BUF_REPLAYED, &drep0, &bytes0));
    f.hologram = ComplexField(cfg.nx, cfg.ny, C, cfg.pitch);
    d2h_widen(f.hologram.data.data(), dholo, n);
    f.replayed = make_parallel<ComplexField>(L, cfg.nx, cfg.ny, C, cfg.pitch);
    for (int l = 0; l < L; ++l)
        d2h_widen(f.replayed[l].data.data(), static_cast<const std::complex<float>*>(drep0) + static_cast<size_t>(l) * n,
                  n);
    lap("hologram+replayed");
    // intensities = intensity(replayed) of the returned fields, literally as
    // pipeline.cpp:26-27 (f64 squares of the widened fp32 replay), formed on the
    // device from the resident replay: no re-upload of the returned fields
    {
        void* drep = nullptr;
        size_t bytes = 0;
        check(holo_frame_buffer(ctx(), HOLO_BUF_REPLAYED, &drep, &bytes));
        const size_t total = static_cast<size_t>(L) * n;
        DevMem dint(sizeof(double) * total);
        check(holo_intensity_widened(ctx(), drep, static_cast<double*>(dint.p), total));
        f.intensities = make_parallel<IntensityImage>(L, cfg.nx, cfg.ny, C, 0.0);
        for (int l = 0; l < L; ++l)
            d2h(f.intensities[l].data.data(), static_cast<const double*>(dint.p) + static_cast<size_t>(l) * n,
                sizeof(double) * n);
    }
    lap("intensities");
    return f;
}

// ------------------------------------------------------------------ HOLOFIELD I/O (field_io.cpp)

namespace {
constexpr char kFieldMagic[16] = {'H', 'O', 'L', 'O', 'F', 'I', 'E', 'L', 'D', 0, 0, 0, 0, 0, 0, 0};
struct FileCloser {
    void operator()(std::FILE* f) const {
        if (f) std::fclose(f);
    }
};
using File = std::unique_ptr<std::FILE, FileCloser>;
static_assert(std::endian::native == std::endian::little, "HOLOFIELD is little endian");
}  // namespace

void write_field(const std::string& path, const ComplexField& f) {
    if (f.w <= 0 || f.h <= 0 || f.c <= 0) throw HoloError("io", "write_field: empty field");
    File fp(std::fopen(path.c_str(), "wb"));
    if (!fp) throw HoloError("io", "cannot open for writing: " + path);
    const std::uint32_t dims[3] = {static_cast<std::uint32_t>(f.w), static_cast<std::uint32_t>(f.h),
                                   static_cast<std::uint32_t>(f.c)};
    if (std::fwrite(kFieldMagic, 1, 16, fp.get()) != 16 || std::fwrite(dims, 4, 3, fp.get()) != 3 ||
        std::fwrite(f.data.data(), sizeof(c64), f.data.size(), fp.get()) != f.data.size() ||
        std::fflush(fp.get()) != 0)
        throw HoloError("io", "short write: " + path);
}

ComplexField read_field(const std::string& path, double pitch) {
    File fp(std::fopen(path.c_str(), "rb"));
    if (!fp) throw HoloError("io", "cannot open: " + path);
    char magic[16];
    if (std::fread(magic, 1, 16, fp.get()) != 16) throw HoloError("io", "truncated header: " + path);
    if (std::memcmp(magic, kFieldMagic, 16) != 0) throw HoloError("io", "bad magic, not a HOLOFIELD file: " + path);
    std::uint32_t dims[3];
    if (std::fread(dims, 4, 3, fp.get()) != 3) throw HoloError("io", "truncated header: " + path);
    if (dims[0] == 0 || dims[1] == 0 || dims[2] == 0 || dims[2] > 64)
        throw HoloError("io", "implausible dimensions in " + path);
    const size_t n = static_cast<size_t>(dims[0]) * dims[1] * dims[2];
    if (n > (1ull << 28)) throw HoloError("io", "field too large in " + path);
    ComplexField f(static_cast<int>(dims[0]), static_cast<int>(dims[1]), static_cast<int>(dims[2]), pitch);
    if (std::fread(f.data.data(), sizeof(c64), n, fp.get()) != n) throw HoloError("io", "truncated payload: " + path);
    return f;
}

// ------------------------------------------------------------------ HOLOSCENE1 I/O (scene_io.cpp:29-95)

namespace {
constexpr char kSceneMagic[10] = {'H', 'O', 'L', 'O', 'S', 'C', 'E', 'N', 'E', '1'};

// the integer value of "key" in a flat JSON object (the header's N and L)
bool json_uint(const std::string& js, const char* key, unsigned long long* out) {
    const std::string k = std::string("\"") + key + "\"";
    size_t p = js.find(k);
    if (p == std::string::npos) return false;
    p = js.find(':', p + k.size());
    if (p == std::string::npos) return false;
    ++p;
    while (p < js.size() && (js[p] == ' ' || js[p] == '\t' || js[p] == '\n' || js[p] == '\r')) ++p;
    if (p >= js.size() || js[p] < '0' || js[p] > '9') return false;
    unsigned long long v = 0;
    while (p < js.size() && js[p] >= '0' && js[p] <= '9') v = v * 10 + static_cast<unsigned>(js[p++] - '0');
    *out = v;
    return true;
}
}  // namespace

void write_scene(const std::string& path, const GaussianScene& s) {
    s.validate();
    // the header as nlohmann::json::dump() writes it (keys sorted)
    const std::string hs =
        "{\"L\":" + std::to_string(s.num_planes) + ",\"N\":" + std::to_string(s.size()) +
        ",\"units\":{\"amplitudes\":\"linear\",\"opacities\":\"logit\",\"phases\":\"rad\",\"plane_logits\":\"logit\","
        "\"positions\":\"m\",\"rotations\":\"unit_quaternion_wxyz\",\"scales\":\"log_m\"}}";
    File fp(std::fopen(path.c_str(), "wb"));
    if (!fp) throw HoloError("io", "cannot open for writing: " + path);
    const std::uint32_t hlen = static_cast<std::uint32_t>(hs.size());
    bool ok = std::fwrite(kSceneMagic, 1, 10, fp.get()) == 10 && std::fwrite(&hlen, 4, 1, fp.get()) == 1 &&
              std::fwrite(hs.data(), 1, hs.size(), fp.get()) == hs.size();
    for (const auto* v : {&s.positions, &s.rotations, &s.log_scales, &s.amplitudes, &s.opacity_logits, &s.phases,
                          &s.plane_logits})
        ok = ok && std::fwrite(v->data(), sizeof(double), v->size(), fp.get()) == v->size();
    if (!ok || std::fflush(fp.get()) != 0) throw HoloError("io", "short write: " + path);
}

GaussianScene read_scene(const std::string& path) {
    File fp(std::fopen(path.c_str(), "rb"));
    if (!fp) throw HoloError("io", "cannot open: " + path);
    char magic[10];
    if (std::fread(magic, 1, 10, fp.get()) != 10) throw HoloError("io", "truncated header: " + path);
    if (std::memcmp(magic, kSceneMagic, 10) != 0) throw HoloError("io", "bad magic, not a HOLOSCENE1 file: " + path);
    std::uint32_t hlen = 0;
    if (std::fread(&hlen, 4, 1, fp.get()) != 1) throw HoloError("io", "truncated header: " + path);
    if (hlen == 0 || hlen > (1u << 20)) throw HoloError("io", "implausible header length in " + path);
    std::string hs(hlen, '\0');
    if (std::fread(hs.data(), 1, hlen, fp.get()) != hlen) throw HoloError("io", "truncated header: " + path);
    unsigned long long n = 0, L = 0;
    if (!json_uint(hs, "N", &n) || !json_uint(hs, "L", &L)) throw HoloError("io", "scene header missing N or L: " + path);
    if (L < 1 || n > (1ull << 26)) throw HoloError("io", "implausible scene dimensions in " + path);
    GaussianScene s;
    s.num_planes = static_cast<int>(L);
    const size_t counts[7] = {n * 3, n * 4, n * 3, n * 3, n, n * 3, n * L};
    std::vector<double>* arrays[7] = {&s.positions, &s.rotations, &s.log_scales, &s.amplitudes,
                                      &s.opacity_logits, &s.phases, &s.plane_logits};
    for (int k = 0; k < 7; ++k) {
        arrays[k]->resize(counts[k]);
        if (std::fread(arrays[k]->data(), sizeof(double), counts[k], fp.get()) != counts[k])
            throw HoloError("io", "truncated payload: " + path);
    }
    s.validate();
    return s;
}

// ------------------------------------------------------------------ losses (losses.cpp, ssim.cpp)

namespace {

void check_stack(const std::vector<IntensityImage>& I, const std::vector<IntensityImage>& I_gt) {  // losses.cpp:11-17
    if (I.size() != I_gt.size() || I.empty()) throw HoloError("config", "focal stacks have different plane counts");
    for (size_t l = 0; l < I.size(); ++l)
        if (I[l].w != I_gt[l].w || I[l].h != I_gt[l].h || I[l].c != I_gt[l].c)
            throw HoloError("config", "focal stack image shapes differ");
    // one batched device call: the planes of a stack share one shape (they always
    // do in the reference's pipeline; mixed shapes are rejected here)
    for (size_t l = 1; l < I.size(); ++l)
        if (I[l].w != I[0].w || I[l].h != I[0].h || I[l].c != I[0].c)
            throw HoloError("config", "focal stack planes must share one image shape");
}

void check_grad(const std::vector<IntensityImage>& I, std::vector<IntensityImage>* grad) {
    if (!grad) return;
    if (grad->size() != I.size()) throw HoloError("config", "loss gradient stack has the wrong plane count");
    for (size_t l = 0; l < I.size(); ++l)
        if ((*grad)[l].data.size() != I[l].data.size()) throw HoloError("config", "loss gradient image shapes differ");
}

// a stack of equal-shape images as one device f64 array [L][C][H][W]
std::unique_ptr<DevMem> upload_stack(const std::vector<IntensityImage>& v) {
    size_t n = 0;
    for (const IntensityImage& im : v) n += im.data.size();
    auto d = std::make_unique<DevMem>(sizeof(double) * n);
    size_t off = 0;
    for (const IntensityImage& im : v) {
        h2d(static_cast<double*>(d->p) + off, im.data.data(), sizeof(double) * im.data.size());
        off += im.data.size();
    }
    return d;
}

void accumulate(std::vector<IntensityImage>* grad, const std::vector<double>& g, double sign = 1.0) {
    size_t off = 0;
    for (IntensityImage& im : *grad) {
        for (size_t i = 0; i < im.data.size(); ++i) im.data[i] += sign * g[off + i];
        off += im.data.size();
    }
}

// the pointwise terms through holo_losses (SSIM left out): value, psnr per plane
double pointwise_loss(const std::vector<IntensityImage>& I, const std::vector<IntensityImage>& I_gt,
                      const std::vector<IntensityImage>* masks, std::vector<IntensityImage>* grad,
                      std::vector<double>* psnr_out) {
    const int L = static_cast<int>(I.size()), C = I[0].c, H = I[0].h, W = I[0].w;
    const auto dI = upload_stack(I), dG = upload_stack(I_gt);
    std::unique_ptr<DevMem> dM;
    if (masks) dM = upload_stack(*masks);
    const size_t n = static_cast<size_t>(L) * C * H * W;
    std::unique_ptr<DevMem> dg;
    if (grad) dg = std::make_unique<DevMem>(sizeof(double) * n);
    const holo_loss_options lo{0.0, 0.0, masks ? 0 : 1};
    holo_loss_breakdown b{};
    std::vector<double> ps(L);
    check(holo_losses(ctx(), static_cast<const double*>(dI->p), static_cast<const double*>(dG->p),
                      dM ? static_cast<const double*>(dM->p) : nullptr, L, C, H, W, &lo, &b, ps.data(),
                      dg ? static_cast<double*>(dg->p) : nullptr));
    if (grad) {
        std::vector<double> g(n);
        d2h(g.data(), dg->p, sizeof(double) * n);
        accumulate(grad, g);
    }
    if (psnr_out) *psnr_out = ps;
    return b.recon;
}

// mean SSIM per plane of equal-shape stacks, and d(mean SSIM_l)/dx_l when asked
std::vector<double> ssim_planes(const std::vector<IntensityImage>& x, const std::vector<IntensityImage>& y,
                                std::vector<double>* grad) {
    const int L = static_cast<int>(x.size()), C = x[0].c, H = x[0].h, W = x[0].w;
    const auto dx = upload_stack(x), dy = upload_stack(y);
    const size_t n = static_cast<size_t>(L) * C * H * W;
    std::unique_ptr<DevMem> dg;
    if (grad) dg = std::make_unique<DevMem>(sizeof(double) * n);
    std::vector<double> s(L);
    check(holo_ssim(ctx(), static_cast<const double*>(dx->p), static_cast<const double*>(dy->p), L, C, H, W, s.data(),
                    dg ? static_cast<double*>(dg->p) : nullptr));
    if (grad) {
        grad->resize(n);
        d2h(grad->data(), dg->p, sizeof(double) * n);
    }
    return s;
}

}  // namespace

double loss_mse(const std::vector<IntensityImage>& I, const std::vector<IntensityImage>& I_gt,
                std::vector<IntensityImage>* grad) {
    check_stack(I, I_gt);
    check_grad(I, grad);
    return pointwise_loss(I, I_gt, nullptr, grad, nullptr);
}

double loss_recon(const std::vector<IntensityImage>& I, const std::vector<IntensityImage>& I_gt,
                  const std::vector<IntensityImage>& masks, std::vector<IntensityImage>* grad) {
    check_stack(I, I_gt);
    check_grad(I, grad);
    if (masks.size() != I.size()) throw HoloError("config", "mask stack has the wrong plane count");
    for (size_t l = 0; l < I.size(); ++l)
        if (masks[l].w != I[l].w || masks[l].h != I[l].h || masks[l].c != 1)
            throw HoloError("config", "masks must be single-channel and match the image size");
    return pointwise_loss(I, I_gt, &masks, grad, nullptr);
}

double loss_ssim(const std::vector<IntensityImage>& I, const std::vector<IntensityImage>& I_gt, double lambda,
                 std::vector<IntensityImage>* grad) {
    check_stack(I, I_gt);
    check_grad(I, grad);
    std::vector<double> gs;
    const std::vector<double> s = ssim_planes(I, I_gt, grad ? &gs : nullptr);
    const double scale = lambda / static_cast<double>(I.size());  // losses.cpp:98-110
    double total = 0.0;
    for (size_t l = 0; l < I.size(); ++l) total += scale * (1.0 - s[l]);
    if (grad) {
        size_t off = 0;
        for (IntensityImage& im : *grad) {
            for (size_t i = 0; i < im.data.size(); ++i) im.data[i] -= scale * gs[off + i];
            off += im.data.size();
        }
    }
    return total;
}

double psnr(const IntensityImage& I, const IntensityImage& I_gt) {
    if (I.w != I_gt.w || I.h != I_gt.h || I.c != I_gt.c) throw HoloError("config", "psnr: image shapes differ");
    std::vector<double> ps;
    pointwise_loss({I}, {I_gt}, nullptr, nullptr, &ps);
    return ps[0];
}

double ssim_mean(const IntensityImage& x, const IntensityImage& y, IntensityImage* grad_x) {
    if (x.w != y.w || x.h != y.h || x.c != y.c) throw HoloError("config", "ssim: image shapes differ");
    if (x.w < 11 || x.h < 11) throw HoloError("config", "ssim needs images at least 11 pixels in each dimension");
    std::vector<double> g;
    const std::vector<double> s = ssim_planes({x}, {y}, grad_x ? &g : nullptr);
    if (grad_x) {
        *grad_x = IntensityImage(x.w, x.h, x.c);
        grad_x->data = std::move(g);
    }
    return s[0];
}

// ------------------------------------------------------------------ total_loss, targets (pipeline.cpp:9-127)

void FocalStackTarget::validate(const WaveConfig& cfg) const {
    if (images.size() != static_cast<size_t>(cfg.num_planes) || masks.size() != images.size())
        throw HoloError("config", "target plane count does not match the wave config");
    for (size_t l = 0; l < images.size(); ++l) {
        if (images[l].w != cfg.nx || images[l].h != cfg.ny || images[l].c != cfg.channels())
            throw HoloError("config", "target image shape does not match the grid");
        if (masks[l].w != cfg.nx || masks[l].h != cfg.ny || masks[l].c != 1)
            throw HoloError("config", "target masks must be single-channel at grid size");
    }
}

LossBreakdown total_loss(const GaussianScene& scene, const CameraView& cam, const WaveConfig& cfg,
                         const FocalStackTarget& target, const PipelineOptions& opt, SceneGradients* grads,
                         PipelineForward* fwd_out) {
    target.validate(cfg);
    check_raster_inputs(scene, cam, cfg);
    if (cfg.channels() != GaussianScene::kChannels)
        throw HoloError("config", "propagate: field does not match the configured grid");
    const holo_scene_arrays sa = scene_arrays(scene);
    check(holo_scene_upload(ctx(), &sa));
    const auto dT = upload_stack(target.images), dM = upload_stack(target.masks);
    const holo_wave w = to_c(cfg);
    const holo_camera c = to_c(cam);
    const holo_raster_settings st = to_c(opt.raster);
    const holo_prop_options po = to_c(opt.prop);
    const holo_loss_options lo{opt.lambda_ssim, opt.lambda_opacity, opt.use_plain_mse ? 1 : 0};
    LossBreakdown out;
    out.psnr.assign(cfg.num_planes, 0.0);
    holo_loss_breakdown b{};
    std::vector<std::unique_ptr<DevMem>> dm;
    holo_scene_grads hg{};
    std::vector<std::vector<double>*> vs;
    if (grads) {
        grads->resize_like(scene);
        vs = {&grads->positions, &grads->rotations, &grads->log_scales, &grads->amplitudes,
              &grads->opacity_logits, &grads->phases, &grads->plane_logits, &grads->mu_screen};
        double** slots[8] = {&hg.positions, &hg.rotations, &hg.log_scales, &hg.amplitudes,
                             &hg.opacity_logits, &hg.phases, &hg.plane_logits, &hg.mu_screen};
        for (int k = 0; k < 8; ++k) {
            dm.push_back(std::make_unique<DevMem>(sizeof(double) * vs[k]->size()));
            *slots[k] = static_cast<double*>(dm[k]->p);
        }
    }
    check(holo_total_loss(ctx(), &c, &w, &st, &po, &lo, static_cast<const double*>(dT->p),
                          static_cast<const double*>(dM->p), &b, out.psnr.data(), grads ? &hg : nullptr));
    out.total = b.total;
    out.recon = b.recon;
    out.ssim = b.ssim;
    out.opacity = b.opacity;
    out.psnr_mean = b.psnr_mean;
    for (size_t k = 0; k < vs.size(); ++k) d2h(vs[k]->data(), dm[k]->p, sizeof(double) * vs[k]->size());
    if (fwd_out) *fwd_out = pipeline_forward(scene, cam, cfg, opt);
    return out;
}

FocalStackTarget make_target_from_scene(const GaussianScene& oracle, const CameraView& cam, const WaveConfig& cfg,
                                        const PipelineOptions& opt) {
    PipelineForward f = pipeline_forward(oracle, cam, cfg, opt);
    FocalStackTarget t;
    t.camera = cam;
    t.images = std::move(f.intensities);
    const int L = cfg.num_planes;
    // the masks (pipeline.cpp:106-124) from the frame's layers still resident on the
    // device (holo_plane_masks), not from the 800 MB of widened host copies
    const size_t P = static_cast<size_t>(cfg.nx) * cfg.ny;
    t.masks = make_parallel<IntensityImage>(L, cfg.nx, cfg.ny, 1, 0.0);
    DevMem dm(sizeof(double) * L * P);
    check(holo_plane_masks(ctx(), static_cast<double*>(dm.p)));
    for (int l = 0; l < L; ++l)
        d2h(t.masks[l].data.data(), static_cast<const double*>(dm.p) + static_cast<size_t>(l) * P, sizeof(double) * P);
    return t;
}

// ------------------------------------------------------------------ optimizer (optimizer.cpp)

double cosine_lr(double base, double floor, long long t, long long total) {
    if (total <= 0 || t >= total) return floor;
    const double phase = kPi * static_cast<double>(t) / static_cast<double>(total);
    return floor + 0.5 * (base - floor) * (1.0 + std::cos(phase));
}

void OptimState::Moments::resize(size_t count) {
    m.assign(count, 0.0);
    v.assign(count, 0.0);
    n.assign(count, 0.0);
    prev_grad.assign(count, 0.0);
}

void OptimState::Moments::remap_rows(const std::vector<int>& src_index, size_t stride) {
    std::vector<double>* arrs[4] = {&m, &v, &n, &prev_grad};
    for (std::vector<double>* a : arrs) {
        std::vector<double> out(src_index.size() * stride, 0.0);
        for (size_t j = 0; j < src_index.size(); ++j) {
            const int src = src_index[j];
            if (src < 0) continue;
            std::copy_n(a->begin() + static_cast<std::ptrdiff_t>(src * stride), stride,
                        out.begin() + static_cast<std::ptrdiff_t>(j * stride));
        }
        a->swap(out);
    }
}

void OptimState::resize_like(const GaussianScene& s) {
    positions.resize(s.positions.size());
    rotations.resize(s.rotations.size());
    log_scales.resize(s.log_scales.size());
    amplitudes.resize(s.amplitudes.size());
    opacities.resize(s.opacity_logits.size());
    phases.resize(s.phases.size());
    plane_logits.resize(s.plane_logits.size());
}

void OptimState::remap(const std::vector<int>& src_index, const GaussianScene& new_scene) {
    positions.remap_rows(src_index, 3);
    rotations.remap_rows(src_index, 4);
    log_scales.remap_rows(src_index, 3);
    amplitudes.remap_rows(src_index, 3);
    opacities.remap_rows(src_index, 1);
    phases.remap_rows(src_index, 3);
    plane_logits.remap_rows(src_index, static_cast<size_t>(new_scene.num_planes));
}

void adaptive_moment_update(std::vector<double>& params, const std::vector<double>& grads, OptimState::Moments& mom,
                            double lr, long long step, const OptimizerConfig& cfg) {
    const size_t n = params.size();
    if (grads.size() != n || mom.m.size() != n || mom.v.size() != n || mom.n.size() != n || mom.prev_grad.size() != n)
        throw HoloError("config", "optimizer: gradient or moment sizes do not match the parameters");
    if (n == 0) return;
    // six f64 arrays through one device call (holo_adaptive_update)
    DevMem d(sizeof(double) * 6 * n);
    double* p = static_cast<double*>(d.p);
    const std::vector<double>* src[6] = {&params, &grads, &mom.m, &mom.v, &mom.n, &mom.prev_grad};
    for (int k = 0; k < 6; ++k) h2d(p + k * n, src[k]->data(), sizeof(double) * n);
    const holo_optimizer_config c{cfg.lr_positions, cfg.lr_rotations, cfg.lr_log_scales, cfg.lr_amplitudes,
                                  cfg.lr_phases,    cfg.lr_opacities, cfg.lr_plane_logits, cfg.beta1,
                                  cfg.beta2,        cfg.beta3,        cfg.eps,             cfg.use_adam ? 1 : 0,
                                  cfg.schedule_total, cfg.lr_floor};
    check(holo_adaptive_update(ctx(), p, p + n, p + 2 * n, p + 3 * n, p + 4 * n, p + 5 * n, n, lr, step, &c));
    std::vector<double>* dst[6] = {&params, nullptr, &mom.m, &mom.v, &mom.n, &mom.prev_grad};
    for (int k = 0; k < 6; ++k)
        if (dst[k]) d2h(dst[k]->data(), p + k * n, sizeof(double) * n);
}

bool optimizer_step(OptimState& st, GaussianScene& scene, const SceneGradients& grads, const OptimizerConfig& cfg) {
    if (grads.positions.size() != scene.positions.size() || grads.plane_logits.size() != scene.plane_logits.size())
        throw HoloError("config", "optimizer: gradient shapes do not match the scene");
    if (st.positions.m.size() != scene.positions.size())
        throw HoloError("config", "optimizer: moment buffers do not match the scene");
    for (const std::vector<double>* g : {&grads.positions, &grads.rotations, &grads.log_scales, &grads.amplitudes,
                                         &grads.opacity_logits, &grads.phases, &grads.plane_logits})
        for (double x : *g)
            if (!std::isfinite(x)) {
                ++st.skipped;
                return false;
            }
    const long long t = st.step;
    ++st.step;
    const double lr_pos = cosine_lr(cfg.lr_positions, cfg.lr_floor, t, cfg.schedule_total);
    const double lr_rho = cosine_lr(cfg.lr_plane_logits, cfg.lr_floor, t, cfg.schedule_total);
    adaptive_moment_update(scene.positions, grads.positions, st.positions, lr_pos, st.step, cfg);
    adaptive_moment_update(scene.rotations, grads.rotations, st.rotations, cfg.lr_rotations, st.step, cfg);
    adaptive_moment_update(scene.log_scales, grads.log_scales, st.log_scales, cfg.lr_log_scales, st.step, cfg);
    adaptive_moment_update(scene.amplitudes, grads.amplitudes, st.amplitudes, cfg.lr_amplitudes, st.step, cfg);
    adaptive_moment_update(scene.opacity_logits, grads.opacity_logits, st.opacities, cfg.lr_opacities, st.step, cfg);
    adaptive_moment_update(scene.phases, grads.phases, st.phases, cfg.lr_phases, st.step, cfg);
    adaptive_moment_update(scene.plane_logits, grads.plane_logits, st.plane_logits, lr_rho, st.step, cfg);
    scene.renormalize();
    return true;
}

// ------------------------------------------------------------------ phase-only conversion (phase_only.cpp)

ComplexField PhaseOnlyHologram::field(double pitch) const {
    ComplexField f(w, h, c, pitch);
    for (size_t i = 0; i < phase.size(); ++i) f.data[i] = std::polar(1.0, phase[i]);
    return f;
}

namespace {

void check_phase_input(const ComplexField& P, const WaveConfig& cfg) {  // phase_only.cpp:22-29
    cfg.validate();
    if (P.w != cfg.nx || P.h != cfg.ny || P.c != cfg.channels())
        throw HoloError("config", "hologram shape does not match the wave config");
    for (const c64& v : P.data)
        if (!std::isfinite(v.real()) || !std::isfinite(v.imag()))
            throw HoloError("numeric", "hologram contains non-finite samples");
}

holo_phase_options to_c(const PhaseOnlyOptions& o) { return {o.lambda_ssim, to_c(o.prop), o.use_adam ? 1 : 0}; }

std::unique_ptr<DevMem> upload_c128(const ComplexField& P) {
    auto d = std::make_unique<DevMem>(sizeof(c64) * P.data.size());
    h2d(d->p, P.data.data(), sizeof(c64) * P.data.size());
    return d;
}

double phase_loss_dev(const DevMem& dP, const std::vector<double>& theta, const WaveConfig& cfg,
                      const PhaseOnlyOptions& opt, std::vector<double>* grad) {
    DevMem dt(sizeof(double) * theta.size());
    h2d(dt.p, theta.data(), sizeof(double) * theta.size());
    std::unique_ptr<DevMem> dg;
    if (grad) dg = std::make_unique<DevMem>(sizeof(double) * theta.size());
    const holo_wave w = to_c(cfg);
    const holo_phase_options po = to_c(opt);
    double loss = 0.0;
    check(holo_phase_only_loss(ctx(), dP.p, static_cast<const double*>(dt.p), &w, &po, &loss,
                               dg ? static_cast<double*>(dg->p) : nullptr));
    if (grad) {
        grad->resize(theta.size());
        d2h(grad->data(), dg->p, sizeof(double) * theta.size());
    }
    return loss;
}

}  // namespace

double phase_only_loss(const ComplexField& P, const std::vector<double>& theta, const WaveConfig& cfg,
                       const PhaseOnlyOptions& opt, std::vector<double>* grad) {
    check_phase_input(P, cfg);
    if (theta.size() != P.data.size()) throw HoloError("config", "phase vector does not match the hologram shape");
    const auto dP = upload_c128(P);
    return phase_loss_dev(*dP, theta, cfg, opt, grad);
}

PhaseOnlyResult convert_phase_only(const ComplexField& P, const WaveConfig& cfg, int iters, double lr,
                                   const PhaseOnlyOptions& opt) {
    check_phase_input(P, cfg);
    if (iters < 0) throw HoloError("config", "iteration count must be non-negative");
    if (lr <= 0.0) throw HoloError("config", "step size must be positive");
    PhaseOnlyResult out;
    out.hologram.w = P.w;
    out.hologram.h = P.h;
    out.hologram.c = P.c;
    std::vector<double> theta(P.data.size());
    for (size_t i = 0; i < theta.size(); ++i) theta[i] = std::arg(P.data[i]);  // the reference's extraction
    const auto dP = upload_c128(P);
    DevMem dt(sizeof(double) * theta.size()), dphase(sizeof(double) * theta.size());
    h2d(dt.p, theta.data(), sizeof(double) * theta.size());
    const holo_wave w = to_c(cfg);
    const holo_phase_options po = to_c(opt);
    out.trace.assign(static_cast<size_t>(iters) + 1, 0.0);
    check(holo_convert_phase_only(ctx(), dP->p, &w, iters, lr, &po, static_cast<const double*>(dt.p),
                                  static_cast<double*>(dphase.p), out.trace.data()));
    out.hologram.phase.resize(theta.size());
    d2h(out.hologram.phase.data(), dphase.p, sizeof(double) * theta.size());
    return out;
}

std::vector<double> phase_gradient_oracle(const ComplexField& P, const std::vector<double>& theta,
                                          const WaveConfig& cfg, const std::vector<size_t>& indices, double fd_step,
                                          const PhaseOnlyOptions& opt) {
    if (cfg.num_planes < 1) throw HoloError("config", "oracle needs at least one depth plane");
    if (cfg.nx > 64 || cfg.ny > 64) throw HoloError("config", "oracle is limited to grids up to 64x64");
    check_phase_input(P, cfg);
    if (theta.size() != P.data.size()) throw HoloError("config", "phase vector does not match the hologram shape");
    if (fd_step <= 0.0) throw HoloError("config", "difference step must be positive");
    std::vector<size_t> idx = indices;
    if (idx.empty()) {
        idx.resize(theta.size());
        for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    }
    const auto dP = upload_c128(P);
    std::vector<double> g(theta.size(), 0.0), probe = theta;
    for (size_t i : idx) {
        if (i >= theta.size()) throw HoloError("config", "sampled phase index out of range");
        probe[i] = theta[i] + fd_step;
        const double up = phase_loss_dev(*dP, probe, cfg, opt, nullptr);
        probe[i] = theta[i] - fd_step;
        const double dn = phase_loss_dev(*dP, probe, cfg, opt, nullptr);
        probe[i] = theta[i];
        g[i] = (up - dn) / (2.0 * fd_step);
    }
    return g;
}

}  // namespace holo
