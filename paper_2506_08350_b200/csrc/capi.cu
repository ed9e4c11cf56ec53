// libholo_cuda C-ABI: context, scene residency, the render orchestration and the
// propagation operators (include/holo_cuda.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "render.h"

using namespace holo_cuda;

namespace {

thread_local std::string g_last_error;

// The largest float not above x: the fp32 alpha clamp never exceeds the
// reference's f64 one (a = min(alpha g, alpha_clamp) <= alpha_clamp and
// T = 1 - a >= 1 - alpha_clamp hold as in test_rasterizer.cpp:327-344).
float float_not_above(double x) {
    float f = static_cast<float>(x);
    if (static_cast<double>(f) > x) f = std::nextafter(f, -INFINITY);
    return f;
}

// intensity (field.cpp:5-14) of complex64 samples widened to f64: the same
// uncontracted std::norm as the f64 operator (k_intensity), so it equals the f64
// intensity of the downloaded, widened field bit for bit
__global__ void k_intensity_widened(const cx<float>* __restrict__ f, double* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double re = f[i].x, im = f[i].y;
        out[i] = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
    }
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return HOLO_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return HOLO_ERR_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return HOLO_ERR_NUMERIC;
    }
}


// WaveConfig::validate (wave_config.cpp:5-16), same messages
void validate_wave(const holo_wave& w) {
    if (w.nx <= 0 || w.ny <= 0) config_error("resolution must be positive");
    if (w.pitch <= 0.0) config_error("pixel pitch must be positive");
    if (w.channels < 1) config_error("at least one wavelength required");
    if (w.channels > HOLO_MAX_CHANNELS) config_error("too many wavelength channels");
    for (int c = 0; c < w.channels; ++c)
        if (w.wavelengths[c] <= 0.0) config_error("wavelengths must be positive");
    if (w.distance <= 0.0) config_error("propagation distance must be positive");
    if (w.volume_depth < 0.0) config_error("volume depth must be non-negative");
    if (w.num_planes < 1) config_error("need at least one depth plane");
    if (w.num_planes > 1 && w.volume_depth <= 0.0) config_error("multiple planes need a positive volume depth");
}

// CameraView::validate (camera.cpp:22-27)
void validate_camera(const holo_camera& c) {
    if (c.width <= 0 || c.height <= 0) config_error("camera resolution must be positive");
    if (c.focal_px <= 0.0) config_error("focal length must be positive");
    for (double v : c.pose)
        if (!std::isfinite(v)) config_error("camera pose must be finite");
}

// plane_positions (wave_config.cpp:18-30)
std::vector<double> plane_positions(const holo_wave& w) {
    validate_wave(w);
    const int L = w.num_planes;
    std::vector<double> z(L);
    if (L == 1) {
        z[0] = w.distance;
        return z;
    }
    const double dz = w.volume_depth / (L - 1);
    const double z0 = w.distance - 0.5 * (L - 1) * dz;
    for (int l = 0; l < L; ++l) z[l] = z0 + l * dz;
    return z;
}

template <class T>
T* buf(holo_ctx* ctx, const char* name, size_t count) {
    return static_cast<T*>(ctx->buffer(name, sizeof(T) * (count ? count : 1)));
}

}  // namespace

// ---------------------------------------------------------------- holo_ctx methods

namespace {

// the guard band of b intact? (synchronises the stream)
bool guard_intact(holo_ctx* ctx, const DevBuf& b) {
    std::vector<unsigned char> h(kGuardBytes);
    HC_CUDA(cudaStreamSynchronize(ctx->stream));
    HC_CUDA(cudaMemcpy(h.data(), static_cast<const unsigned char*>(b.p) + b.guard_at, kGuardBytes,
                       cudaMemcpyDeviceToHost));
    for (unsigned char v : h)
        if (v != kGuardByte) return false;
    return true;
}

}  // namespace

void* holo_ctx::buffer(const std::string& name, size_t bytes) {
    DevBuf& b = scratch[name];
    if (b.bytes < bytes) {
        if (b.p) {
            HC_CUDA(cudaStreamSynchronize(stream));
            if (guard && !guard_intact(this, b))
                throw Error(HOLO_ERR_NUMERIC, "guard band overwritten past scratch buffer '" + name + "'");
            HC_CUDA(cudaFree(b.p));
            b.p = nullptr;
            b.bytes = 0;
            small_cache.clear();  // a freed address may come back for another buffer
        }
        if (guard) {  // exact size, then the guard band
            HC_CUDA(cudaMalloc(&b.p, bytes + kGuardBytes));
            HC_CUDA(cudaMemsetAsync(static_cast<unsigned char*>(b.p) + bytes, kGuardByte, kGuardBytes, stream));
            b.bytes = bytes;
            b.guard_at = bytes;
        } else {
            const size_t want = bytes + bytes / 8;  // headroom for frame-to-frame growth
            HC_CUDA(cudaMalloc(&b.p, want));
            b.bytes = want;
        }
    }
    return b.p;
}

void* holo_ctx::pinned(size_t bytes) {
    if (host_pinned_bytes < bytes) {
        if (host_pinned) {
            HC_CUDA(cudaStreamSynchronize(stream));
            HC_CUDA(cudaFreeHost(host_pinned));
        }
        HC_CUDA(cudaMallocHost(&host_pinned, bytes));
        host_pinned_bytes = bytes;
    }
    return host_pinned;
}

template <class T>
const cx<T>* holo_ctx::twiddle(int n) {
    const auto key = std::make_pair(n, static_cast<int>(sizeof(T)));
    auto it = twiddles.find(key);
    if (it != twiddles.end()) return static_cast<const cx<T>*>(it->second);
    std::vector<cx<T>> h(n);
    const double two_pi = 6.283185307179586476925286766559;
    for (int q = 0; q < n; ++q) {
        const double a = -two_pi * static_cast<double>(q) / static_cast<double>(n);
        h[q] = mk<T>(static_cast<T>(std::cos(a)), static_cast<T>(std::sin(a)));
    }
    void* d = nullptr;
    HC_CUDA(cudaMalloc(&d, sizeof(cx<T>) * n));
    HC_CUDA(cudaMemcpy(d, h.data(), sizeof(cx<T>) * n, cudaMemcpyHostToDevice));
    twiddles[key] = d;
    return static_cast<const cx<T>*>(d);
}
template const cx<float>* holo_ctx::twiddle<float>(int);
template const cx<double>* holo_ctx::twiddle<double>(int);

const double* holo_ctx::freq(int n, double pitch) {
    uint64_t bits;
    std::memcpy(&bits, &pitch, sizeof bits);
    const auto key = std::make_pair(n, bits);
    auto it = freqs.find(key);
    if (it != freqs.end()) return it->second;
    std::vector<double> h(n);
    for (int i = 0; i < n; ++i) {
        const int k = (i < (n + 1) / 2) ? i : i - n;  // freq_at, propagation.cpp:13-16
        h[i] = static_cast<double>(k) / (static_cast<double>(n) * pitch);
    }
    double* d = nullptr;
    HC_CUDA(cudaMalloc(&d, sizeof(double) * n));
    HC_CUDA(cudaMemcpy(d, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    freqs[key] = d;
    return d;
}

namespace {

cudaEvent_t take_event(holo_ctx* ctx) {
    if (!ctx->event_pool.empty()) {
        cudaEvent_t e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    HC_CUDA(cudaEventCreate(&e));
    return e;
}

// async upload of a small host table via a pinned ring slot (no stream stall).
// A table identical to the last one uploaded to the same buffer is not sent again:
// frame after frame the render stream then issues no host-to-device copy, which
// would otherwise queue on the copy engine behind the next frame's scene upload.
void upload_small(holo_ctx* ctx, void* dev, const void* host, size_t bytes) {
    auto hit = ctx->small_cache.find(dev);
    if (hit != ctx->small_cache.end() && hit->second.size() == bytes && std::memcmp(hit->second.data(), host, bytes) == 0)
        return;
    ctx->small_cache[dev].assign(static_cast<const unsigned char*>(host), static_cast<const unsigned char*>(host) + bytes);
    if (bytes > holo_ctx::kRingSlotBytes) {
        HC_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
        HC_CUDA(cudaStreamSynchronize(ctx->stream));
        return;
    }
    if (!ctx->ring) {
        HC_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->ring), holo_ctx::kRingSlots * holo_ctx::kRingSlotBytes));
        for (auto& e : ctx->ring_ev) HC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int s = ctx->ring_next;
    ctx->ring_next = (s + 1) % holo_ctx::kRingSlots;
    if (ctx->ring_used[s]) HC_CUDA(cudaEventSynchronize(ctx->ring_ev[s]));
    unsigned char* slot = ctx->ring + static_cast<size_t>(s) * holo_ctx::kRingSlotBytes;
    std::memcpy(slot, host, bytes);
    HC_CUDA(cudaMemcpyAsync(dev, slot, bytes, cudaMemcpyHostToDevice, ctx->stream));
    HC_CUDA(cudaEventRecord(ctx->ring_ev[s], ctx->stream));
    ctx->ring_used[s] = true;
}

}  // namespace

void holo_ctx::stage_begin() {
    if (!timing) return;
    ev_a = take_event(this);
    HC_CUDA(cudaEventRecord(ev_a, stream));
}

void holo_ctx::stage_end(int stage) {
    if (!timing) return;
    cudaEvent_t b = take_event(this);
    HC_CUDA(cudaEventRecord(b, stream));
    pending.push_back({stage, ev_a, b});
    ++stage_calls[stage];
}

namespace {

void resolve_timing(holo_ctx* ctx) {
    if (ctx->pending.empty()) return;
    HC_CUDA(cudaStreamSynchronize(ctx->stream));
    for (const holo_ctx::Timed& t : ctx->pending) {
        float ms = 0.0f;
        HC_CUDA(cudaEventElapsedTime(&ms, t.a, t.b));
        ctx->stage_ms[t.stage] += ms;
        ctx->event_pool.push_back(t.a);
        ctx->event_pool.push_back(t.b);
    }
    ctx->pending.clear();
}

// Fold the status words of finished asynchronous frames into the context, oldest
// first.  wait_all: block until every pending frame is done; otherwise take the
// finished ones and block only while the ring is full.
void consume_status(holo_ctx* ctx, bool wait_all) {
    while (ctx->status_pending_n > 0) {
        const int slot = ctx->status_order[0];
        const cudaEvent_t ev = ctx->status_events[slot];
        if (wait_all || ctx->status_pending_n == holo_ctx::kStatusSlots) {
            HC_CUDA(cudaEventSynchronize(ev));
        } else {
            const cudaError_t q = cudaEventQuery(ev);
            if (q == cudaErrorNotReady) {
                (void)cudaGetLastError();
                break;
            }
            HC_CUDA(q);
        }
        const unsigned* h = ctx->host_status + slot * holo_ctx::kStatusWords;
        ctx->sticky_flags |= h[0];
        ctx->f_num_valid = h[1];
        ctx->f_max_bucket = h[2];
        ctx->f_E = h[4];
        for (int i = 1; i < ctx->status_pending_n; ++i) ctx->status_order[i - 1] = ctx->status_order[i];
        --ctx->status_pending_n;
    }
}

// Outputs written only by the last pass of a frame: a render waits for their
// in-flight asynchronous downloads just before that pass; any other downloaded
// buffer makes it wait before its first kernel.
constexpr unsigned kLateBufs = (1u << HOLO_BUF_HOLOGRAM) | (1u << HOLO_BUF_REPLAYED) | (1u << HOLO_BUF_INTENSITY);

void wait_downloads(holo_ctx* ctx, int set, unsigned mask) {
    for (int k = 0; k < 2; ++k) {
        if ((set >= 0 && k != set) || !(ctx->out_pending[k] & mask)) continue;
        HC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_out_done[k], 0));
        ctx->out_pending[k] = 0;
    }
}

// device buffer name of a final output in set k
std::string out_name(const char* base, int k) { return k ? std::string(base) + ".1" : std::string(base); }

void fill_info(const holo_ctx* ctx, holo_frame_info* info) {
    *info = holo_frame_info{};
    info->num_entries = ctx->f_E;
    info->tiles_x = ctx->f_tiles_x;
    info->tiles_y = ctx->f_tiles_y;
    info->num_buckets = static_cast<int32_t>(ctx->f_buckets);
    info->max_bucket = static_cast<int32_t>(ctx->f_max_bucket);
    info->num_valid = static_cast<int32_t>(ctx->f_num_valid);
}

// ---------------------------------------------------------------- render internals

struct FrameGeom {
    int W, H, C, L, tile, tiles_x, tiles_y, num_tiles;
    size_t P;
};

FrameGeom check_render(holo_ctx* ctx, const holo_camera& cam, const holo_wave& wave, const holo_raster_settings& st) {
    validate_camera(cam);
    validate_wave(wave);
    if (ctx->scene_planes != wave.num_planes)
        config_error("scene plane count does not match the wave config");  // rasterizer.cpp:144-145
    if (cam.width != wave.nx || cam.height != wave.ny)
        config_error("camera resolution must match the hologram grid");  // rasterizer.cpp:146-147
    if (wave.channels > 3) config_error("propagate: field does not match the configured grid");
    if (st.tile != 8 && st.tile != 16 && st.tile != 32) config_error("render supports tile sizes 8, 16 and 32");
    if (st.soft_assignment && wave.num_planes > 64) config_error("soft plane assignment supports at most 64 planes");
    FrameGeom g;
    g.W = wave.nx;
    g.H = wave.ny;
    g.C = wave.channels;
    g.L = wave.num_planes;
    g.tile = st.tile;
    g.tiles_x = (g.W + g.tile - 1) / g.tile;
    g.tiles_y = (g.H + g.tile - 1) / g.tile;
    g.num_tiles = g.tiles_x * g.tiles_y;
    g.P = static_cast<size_t>(g.W) * g.H;
    return g;
}

// raster stage for planes [pb, pe): preprocess, binning, composite -> "layers"
void raster_planes(holo_ctx* ctx, const holo_camera& cam, const holo_wave& wave, const holo_raster_settings& st,
                   const FrameGeom& g, int pb, int pe, unsigned outputs, holo_frame_info* info) {
    const size_t N = ctx->n;
    const int L = g.L;
    const int nplanes = pe - pb;
    const long long B = static_cast<long long>(nplanes) * g.num_tiles;

    CameraConsts cc;
    host_world_to_cam(cam, cc.wc);
    for (int i = 0; i < 3; ++i) cc.pos[i] = cam.pose[i];
    cc.focal = cam.focal_px;
    cc.ppx = cam.cx >= 0.0 ? cam.cx : cam.width / 2.0;   // camera.hpp:26-27
    cc.ppy = cam.cy >= 0.0 ? cam.cy : cam.height / 2.0;
    const double near_clip = st.near_clip > 0.0 ? st.near_clip : 0.2 * wave.distance;  // rasterizer.hpp:25-27

    const bool want_proj = (outputs & HOLO_OUT_PROJECTED) != 0;
    PreOut pre{};
    pre.rec = buf<GRec>(ctx, "rec", N);
    pre.rect = buf<int4>(ctx, "rect", N);
    pre.count = buf<unsigned>(ctx, "count", N);
    pre.zc = buf<double>(ctx, "zc", N);
    pre.plane = buf<int>(ctx, "plane", N);
    pre.pmask = st.soft_assignment ? buf<unsigned long long>(ctx, "pmask", N) : nullptr;
    pre.rho = (st.soft_assignment || want_proj) ? buf<double>(ctx, "rho", N * L) : nullptr;
    pre.touched = buf<unsigned char>(ctx, "touched", N);
    pre.projected = want_proj ? buf<holo_projected>(ctx, "projected", N) : nullptr;
    // flags, num_valid, max bucket, large / mid bucket counts
    unsigned* misc = buf<unsigned>(ctx, "misc", 8);
    pre.flags = misc;
    pre.num_valid = misc + 1;
    unsigned* bcount = buf<unsigned>(ctx, "bcount", B + 1);
    unsigned* bstart = buf<unsigned>(ctx, "bstart", B + 1);
    HC_CUDA(cudaMemsetAsync(misc, 0, sizeof(unsigned) * 8, ctx->stream));
    HC_CUDA(cudaMemsetAsync(bcount, 0, sizeof(unsigned) * (B + 1), ctx->stream));
    // hard assignment: preprocess counts the buckets and hands out entry slots
    const bool hard = !st.soft_assignment;
    unsigned* bbig = hard ? buf<unsigned>(ctx, "bbig", B + 1) : nullptr;
    if (hard) HC_CUDA(cudaMemsetAsync(bbig, 0, sizeof(unsigned) * (B + 1), ctx->stream));
    pre.slots = hard ? buf<unsigned>(ctx, "slots", static_cast<size_t>(kSlots) * N) : nullptr;
    pre.bcount = bcount;
    pre.bbig = bbig;
    pre.pb = pb;
    pre.pe = pe;
    pre.num_tiles = g.num_tiles;

    const int sk = ctx->scene_cur;  // the scene set this frame reads (only preprocess reads it)
    ctx->f_scene_set = sk;
    if (ctx->scene_wait[sk]) {
        HC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_scene_ready[sk], 0));
        ctx->scene_wait[sk] = false;
    }
    ctx->stage_begin();
    preprocess(ctx, cc, st, near_clip, L, g.tiles_x, g.tiles_y, pre);
    ctx->stage_end(0);
    HC_CUDA(cudaEventRecord(ctx->ev_scene_free[sk], ctx->stream));

    ctx->stage_begin();
    if (!hard) bucket_count(ctx, pre, N, L, pb, pe, g.tiles_x, g.num_tiles, st.soft_assignment, bcount);
    exclusive_scan_u32(ctx, bcount, bstart, B, misc + 2, bbig);
    // pinned status words: flags, num_valid, max bucket, -, E
    unsigned* hp = ctx->host_status + holo_ctx::kStatusSlots * holo_ctx::kStatusWords;
    unsigned capacity;
    if (!ctx->async) {
        // synchronous frame: one host round trip for the entry count and the
        // validation flags, so errors surface from this call like the reference's
        publish_status(ctx, misc, bstart + B, hp);
        HC_CUDA(cudaStreamSynchronize(ctx->stream));
        if (hp[0] & kFlagDegenerateQuat) config_error("degenerate quaternion in scene");  // scene.cpp:27
        if (hp[0] & kFlagNegativeAmp) config_error("amplitudes must be non-negative");    // scene.cpp:30
        capacity = hp[4];
        ctx->e_cap = std::max<size_t>(ctx->e_cap, capacity + capacity / 4);  // headroom for later async frames
    } else {
        // asynchronous frame: entries beyond the reserved capacity are dropped and
        // flagged; holo_ctx_frame_status reports it (and the validation flags)
        if (ctx->e_cap == 0) config_error("asynchronous rendering needs holo_ctx_reserve_entries or a synchronous frame first");
        capacity = static_cast<unsigned>(std::min<size_t>(ctx->e_cap, 0xffffffffu));
    }
    // sort keys are the Gaussians' depth bits, gathered by gidx from the 8 MB zc
    // array (L2-resident) instead of being scattered into a per-entry copy
    const auto* zkey = reinterpret_cast<const unsigned long long*>(pre.zc);
    int* egidx = buf<int>(ctx, "egidx", capacity);
    // emission cursors: soft mode counts again from zero in bcount; hard mode keeps
    // bcount (the small Gaussians' slot counts) and counts the large ones in bbig
    unsigned* cursor = hard ? bbig : bcount;
    HC_CUDA(cudaMemsetAsync(cursor, 0, sizeof(unsigned) * (B + 1), ctx->stream));
    bucket_emit(ctx, pre, N, L, pb, pe, g.tiles_x, g.num_tiles, st.soft_assignment, bstart, cursor, egidx,
                capacity, misc);
    // buckets of <= 128 entries sorted one warp each; the larger ones listed, then
    // sorted on the device (mid-size one warp each, large ones CTA-wide)
    sort_small_buckets(ctx, bstart, B, capacity, zkey, egidx, misc + 3);
    sort_large_buckets(ctx, bstart, B, capacity, zkey, egidx, misc + 3);
    ctx->stage_end(1);

    // composite into [nplanes][C][H][W]
    const bool want_aux = (outputs & HOLO_OUT_AUX) != 0;
    const bool want_lists = (outputs & HOLO_OUT_LISTS) != 0;
    CompositeArgs ca{};
    ca.bstart = bstart;
    ca.zkey = zkey;
    ca.egidx = egidx;
    ca.rec = pre.rec;
    ca.rho = pre.rho;
    ca.L = L;
    ca.C = g.C;
    ca.W = g.W;
    ca.H = g.H;
    ca.tiles_x = g.tiles_x;
    ca.num_tiles = g.num_tiles;
    ca.plane_begin = pb;
    ca.num_buckets = static_cast<int>(B);
    ca.soft = st.soft_assignment;
    ca.write_lists = want_lists ? 1 : 0;
    ca.capacity = capacity;
    ca.term_eps = static_cast<float>(st.term_eps);
    ca.alpha_floor = static_cast<float>(st.alpha_floor);
    ca.alpha_clamp = float_not_above(st.alpha_clamp);
    ca.floor_positive = st.alpha_floor > 0.0 ? 1 : 0;
    ca.layers = buf<cx<float>>(ctx, "layers", static_cast<size_t>(nplanes) * g.C * g.P);
    ca.t_final = want_aux ? buf<float>(ctx, "t_final", static_cast<size_t>(nplanes) * g.P) : nullptr;
    ca.n_contrib = want_aux ? buf<int>(ctx, "n_contrib", static_cast<size_t>(nplanes) * g.P) : nullptr;
    ca.e_last = want_aux ? buf<int>(ctx, "e_last", static_cast<size_t>(nplanes) * g.P) : nullptr;
    ctx->stage_begin();
    composite(ctx, ca, g.tile);
    ctx->stage_end(2);
    if (want_lists) entry_depths(ctx, egidx, pre.zc, buf<double>(ctx, "edepth", capacity), bstart + B, capacity);

    ctx->f_tiles_x = g.tiles_x;
    ctx->f_tiles_y = g.tiles_y;
    ctx->f_buckets = B;
    ctx->f_cap = capacity;
    if (!ctx->async) {
        // flags / counters after the whole raster (overflow cannot happen here)
        publish_status(ctx, misc, bstart + B, hp);
        HC_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->f_E = hp[4];
        ctx->f_num_valid = hp[1];
        ctx->f_max_bucket = hp[2];
        if (info) fill_info(ctx, info);
        return;
    }
    // ring slot for this frame's status (waits for the oldest frame when all are in flight)
    consume_status(ctx, false);
    const int slot = ctx->status_next;
    ctx->status_next = (slot + 1) % holo_ctx::kStatusSlots;
    hp = ctx->host_status + slot * holo_ctx::kStatusWords;
    publish_status(ctx, misc, bstart + B, hp);
    HC_CUDA(cudaEventRecord(ctx->status_events[slot], ctx->stream));
    ctx->status_order[ctx->status_pending_n++] = slot;
    if (info) *info = holo_frame_info{};  // known after holo_ctx_frame_status
}

// The row pass evaluates every plane's transfer function directly (instead of the
// plane-to-plane recurrence) for local band limits or unevenly spaced planes.
bool tf_direct(const std::vector<double>& z, int local) {
    // one plane: the recurrence would cost two phasors per sample (A and Q) for one
    if (local || z.size() <= 1) return true;
    for (size_t l = 2; l < z.size(); ++l) {
        const double d0 = z[1] - z[0], d = z[l] - z[l - 1];
        if (std::fabs(d - d0) > 1e-12 * std::fabs(d0)) return true;
    }
    return false;
}

TfChan* upload_tf(holo_ctx* ctx, const char* name, const holo_wave& wave, const std::vector<double>& z, int w, int h,
                  int local) {
    const std::vector<TfChan> t = make_tf_consts(wave, z.data(), static_cast<int>(z.size()), w, h, local);
    TfChan* d = buf<TfChan>(ctx, name, t.size());
    upload_small(ctx, d, t.data(), sizeof(TfChan) * t.size());
    ctx->tf_host[d] = t;  // the row pass keys its cached tables on these (render_static.cu)
    return d;
}

// ---------------------------------------------------------------- generic operators (any precision)

template <class T>
void op_fft2(holo_ctx* ctx, cx<T>* data, int w, int h, int batch, bool inverse) {
    const T s = inverse ? static_cast<T>(1.0 / (static_cast<double>(w) * h)) : T(1);
    rows_fft<T>(ctx, data, data, w, static_cast<long long>(batch) * h, inverse ? +1 : -1, T(1));
    cols_fft<T>(ctx, data, data, w, h, batch, inverse ? +1 : -1, s);
}

// Spectrum of L layers [L][C][h][w] (row-transformed in place in `work`), S = sum_l H_{z_l} FFT2(U_l).
template <class T>
void spectrum_of_layers(holo_ctx* ctx, const cx<T>* layers, cx<T>* work, cx<T>* spec, int w, int h, int C,
                        const holo_wave& wave, const std::vector<double>& z, int local) {
    const int L = static_cast<int>(z.size());
    rows_fft<T>(ctx, layers, work, w, static_cast<long long>(L) * C * h, -1, T(1));
    const TfChan* tfc = upload_tf(ctx, sizeof(T) == 4 ? "tf_f32" : "tf_f64", wave, z, w, h, local);
    col_spectrum<T>(ctx, work, spec, w, h, C, L, tfc, wave.pitch);
}

// out[o] = IFFT2(M_o S) for outputs o with plane_of[o] (-1: none) -> [O][C][h][w] scaled by 1/(w h)
template <class T>
void replay_from_spectrum(holo_ctx* ctx, const cx<T>* spec, cx<T>* out, int w, int h, int C, const holo_wave& wave,
                          const std::vector<double>& z, const std::vector<int>& plane_of, int local) {
    const int O = static_cast<int>(plane_of.size());
    const TfChan* tfc = upload_tf(ctx, sizeof(T) == 4 ? "tfr_f32" : "tfr_f64", wave, z, w, h, local);
    int* d_plane_of = buf<int>(ctx, sizeof(T) == 4 ? "plane_of_f32" : "plane_of_f64", O);
    upload_small(ctx, d_plane_of, plane_of.data(), sizeof(int) * O);
    col_replay<T>(ctx, spec, out, w, h, C, O, d_plane_of, tfc, wave.pitch);
    rows_fft<T>(ctx, out, out, w, static_cast<long long>(O) * C * h, +1,
                static_cast<T>(1.0 / (static_cast<double>(w) * h)));
}

// propagate (propagation.cpp:93-101) on device fields
template <class T>
void op_propagate(holo_ctx* ctx, const cx<T>* in, cx<T>* out, int w, int h, int C, const holo_wave& wave, double z,
                  const holo_prop_options& prop) {
    validate_wave(wave);
    const int pw = prop.pad2x ? 2 * w : w, ph = prop.pad2x ? 2 * h : h;
    const size_t n = static_cast<size_t>(pw) * ph * C;
    cx<T>* a = buf<cx<T>>(ctx, sizeof(T) == 4 ? "prop_a32" : "prop_a64", n);
    cx<T>* s = buf<cx<T>>(ctx, sizeof(T) == 4 ? "prop_s32" : "prop_s64", n);
    const cx<T>* src = in;
    if (prop.pad2x) {
        pad_field<T>(ctx, in, a, w, h, C);
        src = a;
    }
    const std::vector<double> zs{z};
    spectrum_of_layers<T>(ctx, src, a, s, pw, ph, C, wave, zs, prop.local_band_limit);
    cx<T>* dst = prop.pad2x ? a : out;
    replay_from_spectrum<T>(ctx, s, dst, pw, ph, C, wave, zs, std::vector<int>{-1}, prop.local_band_limit);
    if (prop.pad2x) crop_field<T>(ctx, a, out, w, h, C);
}

// forward_record (propagation.cpp:103-114)
template <class T>
void op_forward_record(holo_ctx* ctx, const cx<T>* layers, int L, cx<T>* holo, const holo_wave& wave,
                       const holo_prop_options& prop) {
    const std::vector<double> z = plane_positions(wave);
    if (L != static_cast<int>(z.size())) config_error("forward_record: layer count does not match num_planes");
    const int w = wave.nx, h = wave.ny, C = wave.channels;
    if (!prop.pad2x) {
        const size_t n = static_cast<size_t>(w) * h * C;
        cx<T>* work = buf<cx<T>>(ctx, sizeof(T) == 4 ? "fr_w32" : "fr_w64", n * L);
        cx<T>* s = buf<cx<T>>(ctx, sizeof(T) == 4 ? "fr_s32" : "fr_s64", n);
        spectrum_of_layers<T>(ctx, layers, work, s, w, h, C, wave, z, prop.local_band_limit);
        replay_from_spectrum<T>(ctx, s, holo, w, h, C, wave, z, std::vector<int>{-1}, prop.local_band_limit);
        return;
    }
    // padded: the crop after every propagate (propagation.cpp:100) keeps the planes separate
    const size_t n = static_cast<size_t>(w) * h * C;
    cx<T>* tmp = buf<cx<T>>(ctx, sizeof(T) == 4 ? "fr_t32" : "fr_t64", n);
    for (int l = 0; l < L; ++l) {
        op_propagate<T>(ctx, layers + n * l, tmp, w, h, C, wave, z[l], prop);
        accumulate<T>(ctx, tmp, holo, n, l == 0);
    }
}

// inverse_propagate (propagation.cpp:116-123)
template <class T>
void op_inverse_propagate(holo_ctx* ctx, const cx<T>* holo, cx<T>* replayed, const holo_wave& wave,
                          const holo_prop_options& prop) {
    const std::vector<double> z = plane_positions(wave);
    const int w = wave.nx, h = wave.ny, C = wave.channels, L = static_cast<int>(z.size());
    const size_t n = static_cast<size_t>(w) * h * C;
    if (!prop.pad2x) {
        cx<T>* s = buf<cx<T>>(ctx, sizeof(T) == 4 ? "ip_s32" : "ip_s64", n);
        HC_CUDA(cudaMemcpyAsync(s, holo, sizeof(cx<T>) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        op_fft2<T>(ctx, s, w, h, C, false);
        std::vector<int> plane_of(L);
        for (int l = 0; l < L; ++l) plane_of[l] = l;
        replay_from_spectrum<T>(ctx, s, replayed, w, h, C, wave, z, plane_of, prop.local_band_limit);
        return;
    }
    for (int l = 0; l < L; ++l) op_propagate<T>(ctx, holo, replayed + n * l, w, h, C, wave, -z[l], prop);
}

void check_dtype(int dtype) {
    if (dtype != HOLO_F32 && dtype != HOLO_F64) throw Error(HOLO_ERR_USAGE, "dtype must be HOLO_F32 or HOLO_F64");
}

}  // namespace

// ================================================================== C-ABI

extern "C" {

const char* holo_last_error(void) { return g_last_error.c_str(); }
int holo_abi_version(void) { return HOLO_CUDA_ABI_VERSION; }

int holo_fft_supported(int n) {
    FftPlan p;
    return make_plan(n, &p) ? 1 : 0;
}

int holo_ctx_create(int device, holo_ctx** out) {
    return guarded([&] {
        require(out != nullptr, HOLO_ERR_USAGE, "holo_ctx_create: null output");
        int count = 0;
        HC_CUDA(cudaGetDeviceCount(&count));
        require(device >= 0 && device < count, HOLO_ERR_USAGE, "holo_ctx_create: no such CUDA device");
        HC_CUDA(cudaSetDevice(device));
        auto* ctx = new holo_ctx();
        ctx->device = device;
        HC_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
        if (const char* gv = std::getenv("HOLO_GUARD")) ctx->guard = gv[0] == '1';
        HC_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
        ctx->stream = ctx->own_stream;
        HC_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->host_status),
                               sizeof(unsigned) * (holo_ctx::kStatusSlots + 1) * holo_ctx::kStatusWords));
        std::memset(ctx->host_status, 0, sizeof(unsigned) * (holo_ctx::kStatusSlots + 1) * holo_ctx::kStatusWords);
        for (auto& e : ctx->status_events) HC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        HC_CUDA(cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking));
        HC_CUDA(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k) {
            HC_CUDA(cudaEventCreateWithFlags(&ctx->ev_scene_ready[k], cudaEventDisableTiming));
            HC_CUDA(cudaEventCreateWithFlags(&ctx->ev_scene_free[k], cudaEventDisableTiming));
        }
        HC_CUDA(cudaEventCreateWithFlags(&ctx->ev_out_src, cudaEventDisableTiming));
        for (auto& e : ctx->ev_out_done) HC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        *out = ctx;
    });
}

int holo_ctx_destroy(holo_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(ctx->copy_in);
        cudaStreamSynchronize(ctx->copy_out);
        for (auto& kv : ctx->scratch) cudaFree(kv.second.p);
        for (auto& kv : ctx->twiddles) cudaFree(kv.second);
        for (auto& kv : ctx->freqs) cudaFree(kv.second);
        for (auto& kv : ctx->tables) cudaFree(kv.second);
        for (auto& set : ctx->scene_sets)
            for (double* p : set.a) cudaFree(p);
        for (int k = 0; k < 2; ++k) {
            cudaEventDestroy(ctx->ev_scene_ready[k]);
            cudaEventDestroy(ctx->ev_scene_free[k]);
        }
        cudaEventDestroy(ctx->ev_out_src);
        for (auto e : ctx->ev_out_done) cudaEventDestroy(e);
        for (int c = 0; c < HOLO_MAX_CHANNELS; ++c) {
            if (ctx->ev_chan_ready[c]) cudaEventDestroy(ctx->ev_chan_ready[c]);
            if (ctx->ev_chan_done[c]) cudaEventDestroy(ctx->ev_chan_done[c]);
        }
        cudaStreamDestroy(ctx->copy_in);
        cudaStreamDestroy(ctx->copy_out);
        if (ctx->host_pinned) cudaFreeHost(ctx->host_pinned);
        if (ctx->host_status) cudaFreeHost(ctx->host_status);
        for (auto e : ctx->status_events)
            if (e) cudaEventDestroy(e);
        for (auto& t : ctx->pending) {
            cudaEventDestroy(t.a);
            cudaEventDestroy(t.b);
        }
        for (auto e : ctx->event_pool) cudaEventDestroy(e);
        if (ctx->ring) {
            cudaFreeHost(ctx->ring);
            for (auto e : ctx->ring_ev) cudaEventDestroy(e);
        }
        cudaStreamDestroy(ctx->own_stream);
        delete ctx;
    });
}

int holo_ctx_set_stream(holo_ctx* ctx, void* stream) {
    return guarded([&] {
        require(ctx != nullptr, HOLO_ERR_USAGE, "null context");
        HC_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->stream = static_cast<cudaStream_t>(stream);
    });
}

int holo_ctx_use_own_stream(holo_ctx* ctx) {
    return guarded([&] {
        require(ctx != nullptr, HOLO_ERR_USAGE, "null context");
        HC_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->stream = ctx->own_stream;
    });
}

void* holo_ctx_get_stream(holo_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

void* holo_ctx_get_copy_stream(holo_ctx* ctx, int which) {
    if (!ctx) return nullptr;
    return static_cast<void*>(which == 0 ? ctx->copy_in : ctx->copy_out);
}

int holo_ctx_synchronize(holo_ctx* ctx) {
    return guarded([&] {
        require(ctx != nullptr, HOLO_ERR_USAGE, "null context");
        HC_CUDA(cudaStreamSynchronize(ctx->stream));
        HC_CUDA(cudaStreamSynchronize(ctx->copy_in));
        HC_CUDA(cudaStreamSynchronize(ctx->copy_out));
        ctx->out_pending[0] = ctx->out_pending[1] = 0;
        consume_status(ctx, true);
    });
}

int holo_ctx_set_async(holo_ctx* ctx, int enable) {
    return guarded([&] {
        require(ctx != nullptr, HOLO_ERR_USAGE, "null context");
        if (!enable) consume_status(ctx, true);
        ctx->async = enable != 0;
    });
}

int holo_ctx_reserve_entries(holo_ctx* ctx, uint64_t entries) {
    return guarded([&] {
        require(ctx != nullptr, HOLO_ERR_USAGE, "null context");
        require(entries < 0xffffffffull, HOLO_ERR_USAGE, "holo_ctx_reserve_entries: at most 2^32 - 2 entries");
        ctx->e_cap = std::max<size_t>(ctx->e_cap, static_cast<size_t>(entries));
    });
}

int holo_ctx_frame_status(holo_ctx* ctx, holo_frame_info* info) {
    return guarded([&] {
        require(ctx != nullptr, HOLO_ERR_USAGE, "null context");
        consume_status(ctx, true);
        if (info) fill_info(ctx, info);
        const unsigned f = ctx->sticky_flags;
        ctx->sticky_flags = 0;
        if (f & kFlagDegenerateQuat) config_error("degenerate quaternion in scene");  // scene.cpp:27
        if (f & kFlagNegativeAmp) config_error("amplitudes must be non-negative");    // scene.cpp:30
        if (f & kFlagOverflow) {
            const std::string m = "asynchronous frame needed " + std::to_string(ctx->f_E) +
                                  " entries but only " + std::to_string(ctx->e_cap) +
                                  " are reserved (holo_ctx_reserve_entries); its outputs are incomplete";
            ctx->e_cap = std::max<size_t>(ctx->e_cap, ctx->f_E + ctx->f_E / 4);
            throw Error(HOLO_ERR_NUMERIC, m);
        }
    });
}

int holo_ctx_enable_timing(holo_ctx* ctx, int enable) {
    return guarded([&] { ctx->timing = enable != 0; });
}

int holo_ctx_stage_times(holo_ctx* ctx, double* ms_out, int* launches_out, int max_stages) {
    return guarded([&] {
        resolve_timing(ctx);
        for (int s = 0; s < max_stages && s < kNumStages; ++s) {
            if (ms_out) ms_out[s] = ctx->stage_ms[s];
            if (launches_out) launches_out[s] = ctx->stage_calls[s];
        }
    });
}

int holo_ctx_reset_timing(holo_ctx* ctx) {
    return guarded([&] {
        resolve_timing(ctx);
        for (int s = 0; s < kNumStages; ++s) {
            ctx->stage_ms[s] = 0.0;
            ctx->stage_calls[s] = 0;
        }
    });
}

uint64_t holo_ctx_launch_count(holo_ctx* ctx) { return ctx ? ctx->launches : 0; }

int holo_ctx_set_guard(holo_ctx* ctx, int enable) {
    return guarded([&] {
        require(ctx != nullptr, HOLO_ERR_USAGE, "null context");
        require(ctx->scratch.empty() || (enable != 0) == ctx->guard, HOLO_ERR_USAGE,
                "holo_ctx_set_guard: set guard mode before the first render");
        ctx->guard = enable != 0;
    });
}

int holo_ctx_check_guards(holo_ctx* ctx) {
    return guarded([&] {
        require(ctx != nullptr, HOLO_ERR_USAGE, "null context");
        require(ctx->guard, HOLO_ERR_USAGE, "holo_ctx_check_guards: guard mode is off");
        HC_CUDA(cudaSetDevice(ctx->device));
        std::string bad;
        for (const auto& kv : ctx->scratch)
            if (kv.second.p && !guard_intact(ctx, kv.second)) bad += (bad.empty() ? "" : ", ") + kv.first;
        if (!bad.empty()) throw Error(HOLO_ERR_NUMERIC, "guard band overwritten past scratch buffer(s): " + bad);
    });
}

static int scene_upload(holo_ctx* ctx, const holo_scene_arrays* s, cudaMemcpyKind kind) {
    return guarded([&] {
        require(ctx && s, HOLO_ERR_USAGE, "null argument");
        if (s->num_planes < 1) config_error("scene needs at least one plane");  // scene.cpp:21
        const size_t n = s->n;
        if (n > 0)
            require(s->positions && s->rotations && s->log_scales && s->amplitudes && s->opacity_logits && s->phases &&
                        s->plane_logits,
                    HOLO_ERR_CONFIG, "scene arrays have inconsistent sizes");
        HC_CUDA(cudaSetDevice(ctx->device));
        const double* src[7] = {s->positions, s->rotations, s->log_scales, s->amplitudes,
                                s->opacity_logits, s->phases, s->plane_logits};
        const size_t count[7] = {3 * n, 4 * n, 3 * n, 3 * n, n, 3 * n, n * static_cast<size_t>(s->num_planes)};
        // fill the set the last render is not reading
        const int k = ctx->scene_cur ^ 1;
        holo_ctx::SceneSet& set = ctx->scene_sets[k];
        bool grow = false;
        for (int a = 0; a < 7; ++a) grow = grow || count[a] > set.cap[a] || !set.a[a];
        if (grow) {
            HC_CUDA(cudaStreamSynchronize(ctx->stream));
            HC_CUDA(cudaStreamSynchronize(ctx->copy_in));
            for (int a = 0; a < 7; ++a) {
                cudaFree(set.a[a]);
                set.a[a] = nullptr;
                HC_CUDA(cudaMalloc(&set.a[a], sizeof(double) * (count[a] ? count[a] : 1)));
                set.cap[a] = count[a];
            }
        }
        if (kind == cudaMemcpyHostToDevice) {
            // copy-in stream: after the last preprocess that read this set
            HC_CUDA(cudaStreamWaitEvent(ctx->copy_in, ctx->ev_scene_free[k], 0));
            for (int a = 0; a < 7; ++a)
                if (count[a])
                    HC_CUDA(cudaMemcpyAsync(set.a[a], src[a], sizeof(double) * count[a], kind, ctx->copy_in));
            HC_CUDA(cudaEventRecord(ctx->ev_scene_ready[k], ctx->copy_in));
            ctx->scene_wait[k] = true;
        } else {
            // device arrays are ordered on the context stream; an earlier host upload
            // into this set may still be in flight
            if (ctx->scene_wait[k]) HC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_scene_ready[k], 0));
            ctx->scene_wait[k] = false;
            for (int a = 0; a < 7; ++a)
                if (count[a])
                    HC_CUDA(cudaMemcpyAsync(set.a[a], src[a], sizeof(double) * count[a], kind, ctx->stream));
        }
        ctx->scene_cur = k;
        double** cur[7] = {&ctx->d_positions, &ctx->d_rotations, &ctx->d_log_scales, &ctx->d_amplitudes,
                           &ctx->d_opacity, &ctx->d_phases, &ctx->d_plane_logits};
        for (int a = 0; a < 7; ++a) *cur[a] = set.a[a];
        ctx->n = n;
        ctx->scene_planes = s->num_planes;
    });
}

int holo_scene_upload(holo_ctx* ctx, const holo_scene_arrays* host) {
    return scene_upload(ctx, host, cudaMemcpyHostToDevice);
}

int holo_scene_upload_device(holo_ctx* ctx, const holo_scene_arrays* dev) {
    return scene_upload(ctx, dev, cudaMemcpyDeviceToDevice);
}

}  // extern "C"

namespace {

std::vector<int> output_planes(unsigned outputs, int np) {
    std::vector<int> plane_of;
    if (outputs & HOLO_OUT_HOLOGRAM) plane_of.push_back(-1);
    if (outputs & (HOLO_OUT_REPLAYED | HOLO_OUT_INTENSITY))
        for (int l = 0; l < np; ++l) plane_of.push_back(l);
    return plane_of;
}

struct OutBufs {
    cx<float>* holo = nullptr;
    cx<float>* rep = nullptr;
    float* ints = nullptr;
};

OutBufs output_buffers(holo_ctx* ctx, unsigned outputs, int np, int C, size_t P) {
    OutBufs o;
    const int k = ctx->out_sel;
    if (outputs & HOLO_OUT_HOLOGRAM)
        o.holo = ctx->out_dest[0] ? static_cast<cx<float>*>(ctx->out_dest[0])
                                  : buf<cx<float>>(ctx, out_name("hologram", k).c_str(), static_cast<size_t>(C) * P);
    if (outputs & HOLO_OUT_REPLAYED)
        o.rep = ctx->out_dest[1]
                    ? static_cast<cx<float>*>(ctx->out_dest[1])
                    : buf<cx<float>>(ctx, out_name("replayed", k).c_str(), static_cast<size_t>(np) * C * P);
    if (outputs & HOLO_OUT_INTENSITY)
        o.ints = ctx->out_dest[2] ? static_cast<float*>(ctx->out_dest[2])
                                  : buf<float>(ctx, out_name("intensity", k).c_str(), static_cast<size_t>(np) * C * P);
    return o;
}

// Second half of the propagation: the hologram and the replayed planes [pb, pe)
// from the spectrum S (forward_record's sum, propagation.cpp:103-114; the replay of
// inverse_propagate, :116-123, reuses S = FFT2(hologram)).
void render_back(holo_ctx* ctx, const holo_wave& wave, const holo_prop_options& po, int pb, int pe,
                 const cx<float>* spec, unsigned outputs) {
    const int W = wave.nx, H = wave.ny, C = wave.channels;
    const size_t P = static_cast<size_t>(W) * H;
    const int np = pe - pb;
    const std::vector<int> plane_of = output_planes(outputs, np);
    ctx->f_outputs |= outputs;
    if (plane_of.empty()) return;
    const std::vector<double> zall = plane_positions(wave);
    std::vector<double> z(zall.begin() + pb, zall.begin() + pe);
    if (z.empty()) z.push_back(0.0);
    const int O = static_cast<int>(plane_of.size());
    const TfChan* tfc = upload_tf(ctx, "tf_replay", wave, z, W, H, po.local_band_limit);
    int* d_plane_of = buf<int>(ctx, "plane_of_replay", O);
    upload_small(ctx, d_plane_of, plane_of.data(), sizeof(int) * O);
    cx<float>* stage = buf<cx<float>>(ctx, "replay_stage", static_cast<size_t>(O) * C * P);
    const OutBufs ob = output_buffers(ctx, outputs, np, C, P);
    const int has_holo = (outputs & HOLO_OUT_HOLOGRAM) ? 1 : 0;
    if (static_render_supported(W, H)) {
        ctx->stage_begin();
        static_row(ctx, kModeReplay, nullptr, const_cast<cx<float>*>(spec), stage, W, H, C, np, has_holo,
                   O - has_holo, tfc, wave.pitch, tf_direct(z, po.local_band_limit));
        ctx->stage_end(5);
        wait_downloads(ctx, ctx->out_sel, ~0u);
        ctx->stage_begin();
        static_col_inv(ctx, stage, W, H, C, O, has_holo, ob.holo, ob.rep, ob.ints);
        ctx->stage_end(6);
        return;
    }
    ctx->stage_begin();
    col_replay<float>(ctx, spec, stage, W, H, C, O, d_plane_of, tfc, wave.pitch);
    ctx->stage_end(5);
    wait_downloads(ctx, ctx->out_sel, ~0u);
    ctx->stage_begin();
    rows_epilogue(ctx, stage, W, H, C, O, has_holo, ob.holo, ob.rep, ob.ints);
    ctx->stage_end(6);
}

// Raster planes [pb, pe) and run the forward half of the propagation.  full: go on
// to the outputs (one GPU owns every plane); otherwise leave the partial spectrum
// S_g in spectrum_out for the caller's all-reduce.
void render_front(holo_ctx* ctx, const holo_camera& cam, const holo_wave& wave, const holo_raster_settings& st,
                  const holo_prop_options& po, int pb, int pe, void* spectrum_out, unsigned outputs,
                  holo_frame_info* info, bool full) {
    const FrameGeom g = check_render(ctx, cam, wave, st);
    require(pb >= 0 && pe <= g.L && pb <= pe, HOLO_ERR_USAGE, "plane range outside [0, num_planes]");
    require(!po.pad2x || full, HOLO_ERR_CONFIG, "plane-sharded rendering does not support pad2x");
    ctx->out_sel ^= 1;  // this frame's final outputs go to the other set
    wait_downloads(ctx, -1, ~kLateBufs);
    if (po.pad2x) wait_downloads(ctx, ctx->out_sel, ~0u);
    ctx->f_L = g.L;
    ctx->f_C = g.C;
    ctx->f_W = g.W;
    ctx->f_H = g.H;
    ctx->f_tiles = g.num_tiles;
    ctx->f_outputs = outputs;
    ctx->f_plane_begin = pb;
    ctx->f_plane_end = pe;
    ctx->f_cam = cam;
    ctx->f_st = st;
    raster_planes(ctx, cam, wave, st, g, pb, pe, outputs, info);
    if (po.pad2x) return;  // holo_render runs the padded operators on the spatial layers
    const int np = pe - pb;
    const std::vector<int> plane_of = output_planes(outputs, np);
    if (full && plane_of.empty()) return;
    cx<float>* spec = (!full && spectrum_out) ? static_cast<cx<float>*>(spectrum_out)
                                              : buf<cx<float>>(ctx, "spectrum", static_cast<size_t>(g.C) * g.P);
    if (np == 0) {
        HC_CUDA(cudaMemsetAsync(spec, 0, sizeof(cx<float>) * g.C * g.P, ctx->stream));
        if (full) render_back(ctx, wave, po, pb, pe, spec, outputs);
        return;
    }
    const std::vector<double> zall = plane_positions(wave);
    const std::vector<double> z(zall.begin() + pb, zall.begin() + pe);
    const TfChan* tfc = upload_tf(ctx, "tf_render", wave, z, g.W, g.H, po.local_band_limit);
    cx<float>* layers = static_cast<cx<float>*>(ctx->buffer("layers", 1));
    const size_t nlay = static_cast<size_t>(np) * g.C * g.P;
    if (static_render_supported(g.W, g.H)) {
        cx<float>* work = layers;
        if (outputs & HOLO_OUT_LAYERS) {  // keep the spatial layers: transform a copy
            work = buf<cx<float>>(ctx, "colwork", nlay);
            HC_CUDA(cudaMemcpyAsync(work, layers, sizeof(cx<float>) * nlay, cudaMemcpyDeviceToDevice, ctx->stream));
        }
        ctx->stage_begin();
        static_col_fwd(ctx, work, g.W, g.H, np * g.C);
        ctx->stage_end(3);
        if (!full) {
            ctx->stage_begin();
            static_row(ctx, kModeSpec, work, spec, nullptr, g.W, g.H, g.C, np, 0, 0, tfc, wave.pitch,
                       tf_direct(z, po.local_band_limit));
            ctx->stage_end(4);
            return;
        }
        const int O = static_cast<int>(plane_of.size());
        const int has_holo = (outputs & HOLO_OUT_HOLOGRAM) ? 1 : 0;
        cx<float>* stage = buf<cx<float>>(ctx, "replay_stage", static_cast<size_t>(O) * g.C * g.P);
        const OutBufs ob = output_buffers(ctx, outputs, np, g.C, g.P);
        ctx->stage_begin();
        static_row(ctx, kModeFull, work, nullptr, stage, g.W, g.H, g.C, np, has_holo, O - has_holo, tfc, wave.pitch,
                   tf_direct(z, po.local_band_limit));
        ctx->stage_end(4);
        wait_downloads(ctx, ctx->out_sel, ~0u);
        ctx->stage_begin();
        static_col_inv(ctx, stage, g.W, g.H, g.C, O, (outputs & HOLO_OUT_HOLOGRAM) ? 1 : 0, ob.holo, ob.rep,
                       ob.ints);
        ctx->stage_end(6);
        return;
    }
    // generic sizes: runtime-planned passes (rows, then the spectrum column pass)
    cx<float>* work = (outputs & HOLO_OUT_LAYERS) ? buf<cx<float>>(ctx, "rowwork", nlay) : layers;
    ctx->stage_begin();
    rows_fft<float>(ctx, layers, work, g.W, static_cast<long long>(np) * g.C * g.H, -1, 1.0f);
    ctx->stage_end(3);
    ctx->stage_begin();
    col_spectrum<float>(ctx, work, spec, g.W, g.H, g.C, np, tfc, wave.pitch);
    ctx->stage_end(4);
    if (full) render_back(ctx, wave, po, pb, pe, spec, outputs);
}

// ---------------------------------------------------------------- backward

// the backward runs on the context's last frame: check that it is the one meant
void check_backward_frame(holo_ctx* ctx, const holo_camera& cam, const holo_wave& wave,
                          const holo_raster_settings& st) {
    validate_wave(wave);
    require((ctx->f_outputs & HOLO_OUT_AUX) != 0, HOLO_ERR_USAGE,
            "backward needs the last render with HOLO_OUT_AUX (t_final, n_contrib)");
    require(ctx->f_W == wave.nx && ctx->f_H == wave.ny && ctx->f_C == wave.channels && ctx->f_L == wave.num_planes,
            HOLO_ERR_USAGE, "backward: wave config differs from the last render's");
    require(std::memcmp(&ctx->f_cam, &cam, sizeof cam) == 0 && std::memcmp(&ctx->f_st, &st, sizeof st) == 0,
            HOLO_ERR_USAGE, "backward: camera or render settings differ from the last render's");
    require(ctx->f_plane_begin == 0 && ctx->f_plane_end == wave.num_planes, HOLO_ERR_USAGE,
            "backward needs a full (unsharded) render");
}

// raster_backward (rasterizer.cpp:332-528) on the last frame's lists and records
void raster_backward(holo_ctx* ctx, const holo_wave& wave, const holo_raster_settings& st,
                     const cx<float>* grad_layers, const holo_scene_grads& grads) {
    consume_status(ctx, true);  // E of an asynchronous frame
    // an overflowed asynchronous frame has truncated lists, and the per-Gaussian
    // entry offsets (the scan of the unclamped counts) would run past egrad
    require(ctx->f_E <= ctx->f_cap && !(ctx->sticky_flags & kFlagOverflow), HOLO_ERR_USAGE,
            ("backward: the last frame overflowed its entry capacity (" + std::to_string(ctx->f_E) + " > " +
             std::to_string(ctx->f_cap) + "); render it again before the backward")
                .c_str());
    const size_t N = ctx->n;
    const int L = wave.num_planes, C = wave.channels;
    const unsigned capacity = ctx->f_cap;
    const size_t E = std::min<uint64_t>(ctx->f_E, capacity);
    const holo_ctx::SceneSet& set = ctx->scene_sets[ctx->f_scene_set];
    const GRec* rec = static_cast<const GRec*>(ctx->buffer("rec", 1));
    BwdRec* brec = buf<BwdRec>(ctx, "bwd_rec", N);
    float* egrad = buf<float>(ctx, "bwd_egrad", E * 13);
    // per-Gaussian offsets into the Gaussian-major entry gradients
    const unsigned* count = static_cast<const unsigned*>(ctx->buffer("count", 1));
    unsigned* goff = buf<unsigned>(ctx, "bwd_goff", N + 1);
    if (N > 0) exclusive_scan_u32(ctx, count, goff, static_cast<long long>(N), nullptr);
    bwd_prep(ctx, N, set.a[3], set.a[5], rec, brec);  // amplitudes, phases of the rendered scene set

    RasterBwdArgs ra{};
    ra.bstart = static_cast<const unsigned*>(ctx->buffer("bstart", 1));
    ra.egidx = static_cast<const int*>(ctx->buffer("egidx", 1));
    ra.rec = rec;
    ra.brec = brec;
    ra.rho = st.soft_assignment ? static_cast<const double*>(ctx->buffer("rho", 1)) : nullptr;
    ra.L = L;
    ra.C = C;
    ra.W = wave.nx;
    ra.H = wave.ny;
    ra.tiles_x = ctx->f_tiles_x;
    ra.num_tiles = ctx->f_tiles;
    ra.plane_begin = 0;
    ra.num_buckets = static_cast<int>(ctx->f_buckets);
    ra.soft = st.soft_assignment;
    ra.capacity = capacity;
    ra.alpha_floor = static_cast<float>(st.alpha_floor);
    ra.alpha_clamp = float_not_above(st.alpha_clamp);
    ra.floor_positive = st.alpha_floor > 0.0 ? 1 : 0;
    ra.grad_layers = grad_layers;
    ra.t_final = static_cast<const float*>(ctx->buffer("t_final", 1));
    ra.n_contrib = static_cast<const int*>(ctx->buffer("n_contrib", 1));
    ra.e_last = static_cast<const int*>(ctx->buffer("e_last", 1));
    ra.goff = goff;
    ra.rect = static_cast<const int4*>(ctx->buffer("rect", 1));
    ra.pmask = st.soft_assignment ? static_cast<const unsigned long long*>(ctx->buffer("pmask", 1)) : nullptr;
    ra.egrad = egrad;
    raster_backward_entries(ctx, ra, st.tile);

    double* outs[8] = {grads.positions, grads.rotations, grads.log_scales, grads.amplitudes,
                       grads.opacity_logits, grads.phases, grads.plane_logits, grads.mu_screen};
    const size_t per[8] = {3, 4, 3, 3, 1, 3, static_cast<size_t>(L), 2};
    for (int k = 0; k < 8; ++k)
        if (outs[k]) HC_CUDA(cudaMemsetAsync(outs[k], 0, sizeof(double) * per[k] * N, ctx->stream));

    GaussBwdArgs ga{};
    ga.n = N;
    ga.L = L;
    ga.pb = 0;
    ga.pe = L;
    ga.num_tiles = ctx->f_tiles;
    ga.tiles_x = ctx->f_tiles_x;
    ga.soft = st.soft_assignment;
    ga.capacity = capacity;
    ga.bstart = ra.bstart;
    ga.egidx = ra.egidx;
    ga.egrad = egrad;
    ga.goff = goff;
    ga.rect = static_cast<const int4*>(ctx->buffer("rect", 1));
    ga.count = static_cast<const unsigned*>(ctx->buffer("count", 1));
    ga.plane = static_cast<const int*>(ctx->buffer("plane", 1));
    ga.pmask = st.soft_assignment ? static_cast<const unsigned long long*>(ctx->buffer("pmask", 1)) : nullptr;
    ga.positions = set.a[0];
    ga.rotations = set.a[1];
    ga.log_scales = set.a[2];
    ga.opacity_logits = set.a[4];
    ga.plane_logits = set.a[6];
    host_world_to_cam(ctx->f_cam, ga.cam.wc);
    for (int i = 0; i < 3; ++i) ga.cam.pos[i] = ctx->f_cam.pose[i];
    ga.cam.focal = ctx->f_cam.focal_px;
    ga.cam.ppx = ctx->f_cam.cx >= 0.0 ? ctx->f_cam.cx : ctx->f_cam.width / 2.0;
    ga.cam.ppy = ctx->f_cam.cy >= 0.0 ? ctx->f_cam.cy : ctx->f_cam.height / 2.0;
    ga.near_clip = st.near_clip > 0.0 ? st.near_clip : 0.2 * wave.distance;  // rasterizer.hpp:25-27
    ga.dilation = st.dilation;
    ga.alpha_floor = st.alpha_floor;
    ga.soft_tau = st.soft_tau;
    ga.ste_tau = st.ste_tau;
    ga.g = grads;
    gauss_backward(ctx, ga);
}

// The adjoint of pipeline_forward's propagation (pipeline.cpp:63-80): the
// recording + replay of the forward, applied to gv = 2 replayed dL/dI.
void adjoint_propagation(holo_ctx* ctx, const holo_wave& wave, const holo_prop_options& po, cx<float>* gv,
                         cx<float>* gholo, cx<float>* glayers) {
    const int W = wave.nx, H = wave.ny, C = wave.channels, L = wave.num_planes;
    const size_t P = static_cast<size_t>(W) * H;
    if (po.pad2x) {  // literal operators, as holo_render does
        op_forward_record<float>(ctx, gv, L, gholo, wave, po);
        op_inverse_propagate<float>(ctx, gholo, glayers, wave, po);
        return;
    }
    const std::vector<double> z = plane_positions(wave);
    const TfChan* tfc = upload_tf(ctx, "tf_bwd", wave, z, W, H, po.local_band_limit);
    const int O = L + 1;  // the hologram, then every plane
    cx<float>* stage = buf<cx<float>>(ctx, "bwd_stage", static_cast<size_t>(O) * C * P);
    if (static_render_supported(W, H)) {
        static_col_fwd(ctx, gv, W, H, L * C);
        static_row(ctx, kModeFull, gv, nullptr, stage, W, H, C, L, 1, L, tfc, wave.pitch,
                   tf_direct(z, po.local_band_limit));
        static_col_inv(ctx, stage, W, H, C, O, 1, gholo, glayers, nullptr);
        return;
    }
    cx<float>* spec = buf<cx<float>>(ctx, "bwd_spectrum", static_cast<size_t>(C) * P);
    rows_fft<float>(ctx, gv, gv, W, static_cast<long long>(L) * C * H, -1, 1.0f);
    col_spectrum<float>(ctx, gv, spec, W, H, C, L, tfc, wave.pitch);
    std::vector<int> plane_of(1, -1);
    for (int l = 0; l < L; ++l) plane_of.push_back(l);
    int* d_plane_of = buf<int>(ctx, "plane_of_bwd", O);
    upload_small(ctx, d_plane_of, plane_of.data(), sizeof(int) * O);
    col_replay<float>(ctx, spec, stage, W, H, C, O, d_plane_of, tfc, wave.pitch);
    rows_epilogue(ctx, stage, W, H, C, O, 1, gholo, glayers, nullptr);
}

// holo_render's body (pipeline_forward, pipeline.cpp:20-29)
void render_full(holo_ctx* ctx, const holo_camera& cam, const holo_wave& wave, const holo_raster_settings& st,
                 const holo_prop_options& po, unsigned outputs, holo_frame_info* info) {
    render_front(ctx, cam, wave, st, po, 0, wave.num_planes, nullptr, outputs, info, true);
    if (!po.pad2x) return;
    // pad2x: the spectrum shortcut does not hold (the crop after each propagate,
    // propagation.cpp:100), so run forward_record / inverse_propagate literally.
    const int W = wave.nx, H = wave.ny, C = wave.channels, L = wave.num_planes;
    const size_t P = static_cast<size_t>(W) * H;
    if (!(outputs & (HOLO_OUT_HOLOGRAM | HOLO_OUT_REPLAYED | HOLO_OUT_INTENSITY))) return;
    const cx<float>* layers = static_cast<const cx<float>*>(ctx->buffer("layers", 1));
    const int k = ctx->out_sel;
    cx<float>* d_holo = (ctx->out_dest[0] && (outputs & HOLO_OUT_HOLOGRAM))
                            ? static_cast<cx<float>*>(ctx->out_dest[0])
                            : buf<cx<float>>(ctx, out_name("hologram", k).c_str(), static_cast<size_t>(C) * P);
    op_forward_record<float>(ctx, layers, L, d_holo, wave, po);
    if (outputs & (HOLO_OUT_REPLAYED | HOLO_OUT_INTENSITY)) {
        cx<float>* d_rep = (ctx->out_dest[1] && (outputs & HOLO_OUT_REPLAYED))
                               ? static_cast<cx<float>*>(ctx->out_dest[1])
                               : buf<cx<float>>(ctx, out_name("replayed", k).c_str(), static_cast<size_t>(L) * C * P);
        op_inverse_propagate<float>(ctx, d_holo, d_rep, wave, po);
        if (outputs & HOLO_OUT_INTENSITY)
            intensity<float>(ctx, d_rep,
                             ctx->out_dest[2] ? static_cast<float*>(ctx->out_dest[2])
                                              : buf<float>(ctx, out_name("intensity", k).c_str(),
                                                           static_cast<size_t>(L) * C * P),
                             static_cast<size_t>(L) * C * P);
    }
}

// holo_pipeline_backward's body (pipeline.cpp:63-91 without the opacity term)
void pipeline_backward(holo_ctx* ctx, const holo_camera& cam, const holo_wave& wave, const holo_raster_settings& st,
                       const holo_prop_options& po, const float* grad_intensities, const holo_scene_grads& grads,
                       void* grad_layers_out, void* grad_hologram_out, const double* grad_intensities64 = nullptr) {
    check_backward_frame(ctx, cam, wave, st);
    require((ctx->f_outputs & HOLO_OUT_REPLAYED) != 0, HOLO_ERR_USAGE,
            "pipeline backward needs the last render with HOLO_OUT_REPLAYED");
    const int W = wave.nx, H = wave.ny, C = wave.channels, L = wave.num_planes;
    const size_t P = static_cast<size_t>(W) * H, n = static_cast<size_t>(L) * C * P;
    const cx<float>* rep = static_cast<const cx<float>*>(ctx->buffer(out_name("replayed", ctx->out_sel), 1));
    cx<float>* gv = buf<cx<float>>(ctx, "bwd_gv", n);
    bwd_seed(ctx, rep, grad_intensities, grad_intensities64, gv, n);
    cx<float>* gl = grad_layers_out ? static_cast<cx<float>*>(grad_layers_out) : buf<cx<float>>(ctx, "bwd_glayers", n);
    cx<float>* gh = grad_hologram_out ? static_cast<cx<float>*>(grad_hologram_out)
                                      : buf<cx<float>>(ctx, "bwd_gholo", static_cast<size_t>(C) * P);
    adjoint_propagation(ctx, wave, po, gv, gh, gl);
    raster_backward(ctx, wave, st, gl, grads);
}

}  // namespace

// ---------------------------------------------------------------- plane-sharded frames, channel by channel
// (the group renderer in group.cu; declared in render.h)
namespace holo_cuda {

void render_whole(holo_ctx* ctx, const holo_camera& cam, const holo_wave& wave, const holo_raster_settings& st,
                  const holo_prop_options& po, unsigned outputs, holo_frame_info* info) {
    render_full(ctx, cam, wave, st, po, outputs, info);
}

void chan_events(holo_ctx* ctx) {
    for (int c = 0; c < HOLO_MAX_CHANNELS; ++c) {
        if (!ctx->ev_chan_ready[c]) HC_CUDA(cudaEventCreateWithFlags(&ctx->ev_chan_ready[c], cudaEventDisableTiming));
        if (!ctx->ev_chan_done[c]) HC_CUDA(cudaEventCreateWithFlags(&ctx->ev_chan_done[c], cudaEventDisableTiming));
    }
}

// Raster planes [pb, pe), then the partial spectrum S_g channel by channel into
// spec ([C][H][W]); ev_chan_ready[c] marks channel c complete on the context
// stream, so the sum over the plane group can start on channel c while the
// row pass of channel c + 1 runs.
void shard_front(holo_ctx* ctx, const holo_camera& cam, const holo_wave& wave, const holo_raster_settings& st,
                 const holo_prop_options& po, int pb, int pe, unsigned outputs, cx<float>* spec,
                 holo_frame_info* info) {
    const FrameGeom g = check_render(ctx, cam, wave, st);
    require(pb >= 0 && pe <= g.L && pb <= pe, HOLO_ERR_USAGE, "plane range outside [0, num_planes]");
    require(!po.pad2x, HOLO_ERR_CONFIG, "plane-sharded rendering does not support pad2x");
    chan_events(ctx);
    ctx->out_sel ^= 1;
    wait_downloads(ctx, -1, ~kLateBufs);
    ctx->f_L = g.L;
    ctx->f_C = g.C;
    ctx->f_W = g.W;
    ctx->f_H = g.H;
    ctx->f_tiles = g.num_tiles;
    ctx->f_outputs = outputs;
    ctx->f_plane_begin = pb;
    ctx->f_plane_end = pe;
    ctx->f_cam = cam;
    ctx->f_st = st;
    raster_planes(ctx, cam, wave, st, g, pb, pe, outputs, info);
    const int np = pe - pb;
    auto all_ready = [&] {
        HC_CUDA(cudaEventRecord(ctx->ev_chan_ready[0], ctx->stream));
        for (int c = 1; c < g.C; ++c) HC_CUDA(cudaEventRecord(ctx->ev_chan_ready[c], ctx->stream));
    };
    if (np == 0) {
        HC_CUDA(cudaMemsetAsync(spec, 0, sizeof(cx<float>) * g.C * g.P, ctx->stream));
        all_ready();
        return;
    }
    const std::vector<double> zall = plane_positions(wave);
    const std::vector<double> z(zall.begin() + pb, zall.begin() + pe);
    const TfChan* tfc = upload_tf(ctx, "tf_render", wave, z, g.W, g.H, po.local_band_limit);
    cx<float>* layers = static_cast<cx<float>*>(ctx->buffer("layers", 1));
    const size_t nlay = static_cast<size_t>(np) * g.C * g.P;
    if (static_render_supported(g.W, g.H)) {
        cx<float>* work = layers;
        if (outputs & HOLO_OUT_LAYERS) {
            work = buf<cx<float>>(ctx, "colwork", nlay);
            HC_CUDA(cudaMemcpyAsync(work, layers, sizeof(cx<float>) * nlay, cudaMemcpyDeviceToDevice, ctx->stream));
        }
        ctx->stage_begin();
        static_col_fwd(ctx, work, g.W, g.H, np * g.C);
        ctx->stage_end(3);
        for (int c = 0; c < g.C; ++c) {
            ctx->stage_begin();
            static_row(ctx, kModeSpec, work, spec, nullptr, g.W, g.H, g.C, np, 0, 0, tfc, wave.pitch,
                       tf_direct(z, po.local_band_limit), c, 1);
            ctx->stage_end(4);
            HC_CUDA(cudaEventRecord(ctx->ev_chan_ready[c], ctx->stream));
        }
        return;
    }
    cx<float>* work = (outputs & HOLO_OUT_LAYERS) ? buf<cx<float>>(ctx, "rowwork", nlay) : layers;
    ctx->stage_begin();
    rows_fft<float>(ctx, layers, work, g.W, static_cast<long long>(np) * g.C * g.H, -1, 1.0f);
    ctx->stage_end(3);
    ctx->stage_begin();
    col_spectrum<float>(ctx, work, spec, g.W, g.H, g.C, np, tfc, wave.pitch);
    ctx->stage_end(4);
    all_ready();
}

// From the summed spectrum: for each channel (after ev_chan_done[c]) the replay of
// planes [pb, pe) and, for the channels in holo_mask, the hologram channel.
void shard_back(holo_ctx* ctx, const holo_wave& wave, const holo_prop_options& po, int pb, int pe,
                const cx<float>* spec, unsigned outputs, unsigned holo_mask) {
    const int W = wave.nx, H = wave.ny, C = wave.channels;
    const size_t P = static_cast<size_t>(W) * H;
    const int np = pe - pb;
    if (!(outputs & HOLO_OUT_HOLOGRAM)) holo_mask = 0;
    holo_mask &= (C >= 32 ? ~0u : ((1u << C) - 1u));
    const unsigned outs = (outputs & ~HOLO_OUT_HOLOGRAM) | (holo_mask ? HOLO_OUT_HOLOGRAM : 0u);
    const std::vector<int> plane_of = output_planes(outs, np);
    ctx->f_outputs |= outs;
    if (plane_of.empty()) {
        for (int c = 0; c < C; ++c) HC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_chan_done[c], 0));
        return;
    }
    const std::vector<double> zall = plane_positions(wave);
    std::vector<double> z(zall.begin() + pb, zall.begin() + pe);
    if (z.empty()) z.push_back(0.0);
    const int O = static_cast<int>(plane_of.size());
    const int hh = holo_mask ? 1 : 0;  // stage slot 0 holds the hologram when any channel is formed here
    const int nrep = O - hh;
    const TfChan* tfc = upload_tf(ctx, "tf_replay", wave, z, W, H, po.local_band_limit);
    cx<float>* stage = buf<cx<float>>(ctx, "replay_stage", static_cast<size_t>(O) * C * P);
    const OutBufs ob = output_buffers(ctx, outs, np, C, P);
    if (static_render_supported(W, H)) {
        for (int c = 0; c < C; ++c) {
            HC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_chan_done[c], 0));
            const int own = (holo_mask >> c) & 1u;
            // a channel whose hologram is formed elsewhere skips stage slot 0
            cx<float>* st_c = stage + static_cast<size_t>(hh && !own ? 1 : 0) * C * P;
            ctx->stage_begin();
            static_row(ctx, kModeReplay, nullptr, const_cast<cx<float>*>(spec), st_c, W, H, C, np, own, nrep, tfc,
                       wave.pitch, tf_direct(z, po.local_band_limit), c, 1);
            ctx->stage_end(5);
        }
        wait_downloads(ctx, ctx->out_sel, ~0u);
        for (int c = 0; c < C; ++c) {
            const int own = (holo_mask >> c) & 1u;
            const cx<float>* st_c = stage + static_cast<size_t>(hh && !own ? 1 : 0) * C * P;
            ctx->stage_begin();
            static_col_inv(ctx, st_c, W, H, C, nrep + own, own, ob.holo, ob.rep, ob.ints, c, 1);
            ctx->stage_end(6);
        }
        return;
    }
    for (int c = 0; c < C; ++c) HC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_chan_done[c], 0));
    int* d_plane_of = buf<int>(ctx, "plane_of_replay", O);
    upload_small(ctx, d_plane_of, plane_of.data(), sizeof(int) * O);
    ctx->stage_begin();
    col_replay<float>(ctx, spec, stage, W, H, C, O, d_plane_of, tfc, wave.pitch);
    ctx->stage_end(5);
    wait_downloads(ctx, ctx->out_sel, ~0u);
    ctx->stage_begin();
    rows_epilogue(ctx, stage, W, H, C, O, hh, ob.holo, ob.rep, ob.ints);
    ctx->stage_end(6);
}

// Keep only the Gaussians whose hard plane lies in [pb, pe) (scene_ops.cu), in
// order: the subset goes to the other scene set, which becomes current.
void scene_restrict_planes(holo_ctx* ctx, int pb, int pe) {
    const int src_k = ctx->scene_cur, dst_k = src_k ^ 1;
    holo_ctx::SceneSet& src = ctx->scene_sets[src_k];
    holo_ctx::SceneSet& dst = ctx->scene_sets[dst_k];
    const size_t n = ctx->n;
    const int L = ctx->scene_planes;
    if (ctx->scene_wait[src_k]) {  // a host upload into the source set may be in flight
        HC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_scene_ready[src_k], 0));
        ctx->scene_wait[src_k] = false;
    }
    if (ctx->scene_wait[dst_k]) {
        HC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_scene_ready[dst_k], 0));
        ctx->scene_wait[dst_k] = false;
    }
    const size_t count[7] = {3 * n, 4 * n, 3 * n, 3 * n, n, 3 * n, n * static_cast<size_t>(L)};
    for (int a = 0; a < 7; ++a)
        if (count[a] > dst.cap[a] || !dst.a[a]) {
            HC_CUDA(cudaStreamSynchronize(ctx->stream));
            cudaFree(dst.a[a]);
            dst.a[a] = nullptr;
            HC_CUDA(cudaMalloc(&dst.a[a], sizeof(double) * (count[a] ? count[a] : 1)));
            dst.cap[a] = count[a];
        }
    const double* sp[7];
    double* dp[7];
    for (int a = 0; a < 7; ++a) {
        sp[a] = src.a[a];
        dp[a] = dst.a[a];
    }
    const size_t kept = scene_keep_planes(ctx, sp, dp, n, L, pb, pe);
    ctx->scene_cur = dst_k;
    double** cur[7] = {&ctx->d_positions, &ctx->d_rotations, &ctx->d_log_scales, &ctx->d_amplitudes,
                       &ctx->d_opacity, &ctx->d_phases, &ctx->d_plane_logits};
    for (int a = 0; a < 7; ++a) *cur[a] = dst.a[a];
    ctx->n = kept;
}

void set_last_error(const char* msg) { g_last_error = msg; }

// destination of the current frame's hologram (the caller's or the context set)
cx<float>* frame_hologram(holo_ctx* ctx, int C, size_t P) {
    if (ctx->out_dest[0]) return static_cast<cx<float>*>(ctx->out_dest[0]);
    return buf<cx<float>>(ctx, out_name("hologram", ctx->out_sel).c_str(), static_cast<size_t>(C) * P);
}

// The current scene of `from` (same device) copied into `to`, ordered after
// everything enqueued on from's stream.
void scene_replicate(holo_ctx* from, holo_ctx* to) {
    cudaEvent_t ev = nullptr;
    HC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    const int k = from->scene_cur;
    if (from->scene_wait[k]) {
        HC_CUDA(cudaStreamWaitEvent(from->stream, from->ev_scene_ready[k], 0));
        from->scene_wait[k] = false;
    }
    HC_CUDA(cudaEventRecord(ev, from->stream));
    HC_CUDA(cudaStreamWaitEvent(to->stream, ev, 0));
    HC_CUDA(cudaEventDestroy(ev));
    const holo_ctx::SceneSet& s = from->scene_sets[k];
    holo_scene_arrays arr{};
    arr.n = from->n;
    arr.num_planes = from->scene_planes;
    arr.positions = s.a[0];
    arr.rotations = s.a[1];
    arr.log_scales = s.a[2];
    arr.amplitudes = s.a[3];
    arr.opacity_logits = s.a[4];
    arr.phases = s.a[5];
    arr.plane_logits = s.a[6];
    if (holo_scene_upload_device(to, &arr) != HOLO_OK) throw Error(HOLO_ERR_CUDA, holo_last_error());
}

}  // namespace holo_cuda

extern "C" {

int holo_raster_backward(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave,
                         const holo_raster_settings* settings, const void* grad_layers, holo_scene_grads* grads) {
    return guarded([&] {
        require(ctx && cam && wave && settings && grad_layers && grads, HOLO_ERR_USAGE, "null argument");
        HC_CUDA(cudaSetDevice(ctx->device));
        check_backward_frame(ctx, *cam, *wave, *settings);
        raster_backward(ctx, *wave, *settings, static_cast<const cx<float>*>(grad_layers), *grads);
    });
}

int holo_pipeline_backward(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave,
                           const holo_raster_settings* settings, const holo_prop_options* prop,
                           const void* grad_intensities, holo_scene_grads* grads, void* grad_layers_out,
                           void* grad_hologram_out) {
    return guarded([&] {
        require(ctx && cam && wave && settings && grad_intensities && grads, HOLO_ERR_USAGE, "null argument");
        HC_CUDA(cudaSetDevice(ctx->device));
        const holo_prop_options po = prop ? *prop : holo_prop_options{0, 0};
        pipeline_backward(ctx, *cam, *wave, *settings, po, static_cast<const float*>(grad_intensities), *grads,
                          grad_layers_out, grad_hologram_out);
    });
}

int holo_brute_force_forward(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave,
                             const holo_raster_settings* settings) {
    return guarded([&] {
        require(ctx && cam && wave && settings, HOLO_ERR_USAGE, "null argument");
        HC_CUDA(cudaSetDevice(ctx->device));
        const holo_prop_options po{0, 0};
        // the tiled raster supplies the projections, records and plane weights
        render_full(ctx, *cam, *wave, *settings, po, HOLO_OUT_LAYERS | HOLO_OUT_PROJECTED, nullptr);
        const size_t N = ctx->n;
        const int L = wave->num_planes, C = wave->channels;
        std::vector<holo_projected> proj(N);
        if (N) {
            HC_CUDA(cudaMemcpyAsync(proj.data(), ctx->buffer("projected", 1), sizeof(holo_projected) * N,
                                    cudaMemcpyDeviceToHost, ctx->stream));
            HC_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        // global front-to-back order over every valid Gaussian (rasterizer.cpp:280-288)
        std::vector<int> order;
        for (size_t i = 0; i < N; ++i)
            if (proj[i].valid) order.push_back(static_cast<int>(i));
        std::sort(order.begin(), order.end(), [&](int a, int b) {
            if (proj[a].zc != proj[b].zc) return proj[a].zc < proj[b].zc;
            return a < b;
        });
        int* d_order = buf<int>(ctx, "brute_order", order.size() + 1);
        if (!order.empty())
            HC_CUDA(cudaMemcpyAsync(d_order, order.data(), sizeof(int) * order.size(), cudaMemcpyHostToDevice,
                                    ctx->stream));
        const size_t P = static_cast<size_t>(wave->nx) * wave->ny;
        cx<float>* layers = buf<cx<float>>(ctx, "layers", static_cast<size_t>(L) * C * P);
        brute_force(ctx, static_cast<const GRec*>(ctx->buffer("rec", 1)), d_order, static_cast<int>(order.size()),
                    static_cast<const int*>(ctx->buffer("plane", 1)),
                    settings->soft_assignment ? static_cast<const double*>(ctx->buffer("rho", 1)) : nullptr, L, C,
                    wave->nx, wave->ny, settings->tile, settings->soft_assignment != 0, 1.0 > settings->plane_eps,
                    static_cast<float>(settings->alpha_floor), settings->alpha_floor > 0.0,
                    float_not_above(settings->alpha_clamp), layers);
        HC_CUDA(cudaStreamSynchronize(ctx->stream));  // order lives on the host stack
    });
}

int holo_render_begin(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave,
                      const holo_raster_settings* settings, const holo_prop_options* prop, int plane_begin,
                      int plane_end, void* spectrum_out, unsigned outputs, holo_frame_info* info) {
    return guarded([&] {
        require(ctx && cam && wave && settings, HOLO_ERR_USAGE, "null argument");
        HC_CUDA(cudaSetDevice(ctx->device));
        const holo_prop_options po = prop ? *prop : holo_prop_options{0, 0};
        render_front(ctx, *cam, *wave, *settings, po, plane_begin, plane_end, spectrum_out, outputs, info, false);
    });
}

int holo_render_end(holo_ctx* ctx, const holo_wave* wave, const holo_prop_options* prop, int plane_begin,
                    int plane_end, const void* spectrum, unsigned outputs) {
    return guarded([&] {
        require(ctx && wave, HOLO_ERR_USAGE, "null argument");
        HC_CUDA(cudaSetDevice(ctx->device));
        validate_wave(*wave);
        const holo_prop_options po = prop ? *prop : holo_prop_options{0, 0};
        require(!po.pad2x, HOLO_ERR_CONFIG, "plane-sharded rendering does not support pad2x");
        require(plane_begin >= 0 && plane_end <= wave->num_planes && plane_begin <= plane_end, HOLO_ERR_USAGE,
                "plane range outside [0, num_planes]");
        const cx<float>* spec = spectrum ? static_cast<const cx<float>*>(spectrum)
                                         : static_cast<const cx<float>*>(ctx->buffer("spectrum", 1));
        render_back(ctx, *wave, po, plane_begin, plane_end, spec, outputs);
    });
}

int holo_render(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave, const holo_raster_settings* settings,
                const holo_prop_options* prop, unsigned outputs, holo_frame_info* info) {
    return guarded([&] {
        require(ctx && cam && wave && settings, HOLO_ERR_USAGE, "null argument");
        HC_CUDA(cudaSetDevice(ctx->device));
        const holo_prop_options po = prop ? *prop : holo_prop_options{0, 0};
        render_full(ctx, *cam, *wave, *settings, po, outputs, info);
    });
}

int holo_frame_buffer(holo_ctx* ctx, int which, void** dev_ptr, size_t* bytes) {
    return guarded([&] {
        require(ctx != nullptr, HOLO_ERR_USAGE, "null context");
        const size_t P = static_cast<size_t>(ctx->f_W) * ctx->f_H;
        const size_t np = static_cast<size_t>(ctx->f_plane_end - ctx->f_plane_begin);
        const size_t C = static_cast<size_t>(ctx->f_C);
        const size_t B = np * ctx->f_tiles;
        std::string name;
        size_t sz = 0;
        if (which == HOLO_BUF_ENTRY_GIDX || which == HOLO_BUF_ENTRY_DEPTH)
            consume_status(ctx, true);  // E of an asynchronous frame
        const size_t E = std::min<uint64_t>(ctx->f_E, ctx->f_cap);
        switch (which) {
            case HOLO_BUF_LAYERS: name = "layers"; sz = np * C * P * 8; break;
            case HOLO_BUF_HOLOGRAM: name = out_name("hologram", ctx->out_sel); sz = C * P * 8; break;
            case HOLO_BUF_REPLAYED: name = out_name("replayed", ctx->out_sel); sz = np * C * P * 8; break;
            case HOLO_BUF_INTENSITY: name = out_name("intensity", ctx->out_sel); sz = np * C * P * 4; break;
            case HOLO_BUF_T_FINAL: name = "t_final"; sz = np * P * 4; break;
            case HOLO_BUF_N_CONTRIB: name = "n_contrib"; sz = np * P * 4; break;
            case HOLO_BUF_ENTRY_GIDX: name = "egidx"; sz = E * 4; break;
            case HOLO_BUF_ENTRY_DEPTH: name = "edepth"; sz = E * 8; break;
            case HOLO_BUF_BUCKET_START: name = "bstart"; sz = (B + 1) * 4; break;
            case HOLO_BUF_PROJECTED: name = "projected"; sz = ctx->n * sizeof(holo_projected); break;
            case HOLO_BUF_RHO: name = "rho"; sz = ctx->n * static_cast<size_t>(ctx->f_L) * 8; break;
            case HOLO_BUF_TOUCHED: name = "touched"; sz = ctx->n; break;
            case HOLO_BUF_SPECTRUM: name = "spectrum"; sz = C * P * 8; break;
            default: throw Error(HOLO_ERR_USAGE, "unknown buffer id");
        }
        auto it = ctx->scratch.find(name);
        if (it == ctx->scratch.end() || it->second.bytes < sz)
            throw Error(HOLO_ERR_USAGE, std::string("buffer not produced by the last render: ") + name);
        if (dev_ptr) *dev_ptr = it->second.p;
        if (bytes) *bytes = sz;
    });
}

int holo_frame_download(holo_ctx* ctx, int which, void* host, size_t bytes) {
    void* d = nullptr;
    size_t sz = 0;
    int rc = holo_frame_buffer(ctx, which, &d, &sz);
    if (rc) return rc;
    return guarded([&] {
        require(bytes == sz, HOLO_ERR_USAGE, "holo_frame_download: size mismatch");
        HC_CUDA(cudaMemcpyAsync(host, d, sz, cudaMemcpyDeviceToHost, ctx->stream));
        HC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int holo_frame_download_async(holo_ctx* ctx, int which, void* host, size_t bytes) {
    void* d = nullptr;
    size_t sz = 0;
    int rc = holo_frame_buffer(ctx, which, &d, &sz);
    if (rc) return rc;
    return guarded([&] {
        require(bytes == sz, HOLO_ERR_USAGE, "holo_frame_download_async: size mismatch");
        // copy-out stream, after the frame work enqueued so far; the next render
        // waits for it before overwriting the buffer (wait_downloads)
        HC_CUDA(cudaEventRecord(ctx->ev_out_src, ctx->stream));
        HC_CUDA(cudaStreamWaitEvent(ctx->copy_out, ctx->ev_out_src, 0));
        HC_CUDA(cudaMemcpyAsync(host, d, sz, cudaMemcpyDeviceToHost, ctx->copy_out));
        const int k = ((1u << which) & kLateBufs) ? ctx->out_sel : 0;  // single-buffered ids count in set 0
        HC_CUDA(cudaEventRecord(ctx->ev_out_done[k], ctx->copy_out));
        ctx->out_pending[k] |= 1u << which;
    });
}

int holo_fft2(holo_ctx* ctx, void* data, int w, int h, int batch, int inverse, int dtype) {
    return guarded([&] {
        require(ctx && data, HOLO_ERR_USAGE, "null argument");
        check_dtype(dtype);
        require(w > 0 && h > 0 && batch >= 0, HOLO_ERR_CONFIG, "fft2: dimensions must be positive");
        if (dtype == HOLO_F32)
            op_fft2<float>(ctx, static_cast<cx<float>*>(data), w, h, batch, inverse != 0);
        else
            op_fft2<double>(ctx, static_cast<cx<double>*>(data), w, h, batch, inverse != 0);
    });
}

int holo_transfer_function(holo_ctx* ctx, const holo_wave* wave, double z, const holo_prop_options* prop, void* out,
                           int dtype) {
    return guarded([&] {
        require(ctx && wave && out, HOLO_ERR_USAGE, "null argument");
        check_dtype(dtype);
        validate_wave(*wave);
        const holo_prop_options po = prop ? *prop : holo_prop_options{0, 0};
        const int w = po.pad2x ? 2 * wave->nx : wave->nx, h = po.pad2x ? 2 * wave->ny : wave->ny;
        const std::vector<double> zs{z};
        const TfChan* tfc = upload_tf(ctx, "tf_op", *wave, zs, w, h, po.local_band_limit);
        if (dtype == HOLO_F32)
            transfer_function<float>(ctx, static_cast<cx<float>*>(out), w, h, wave->channels, tfc, wave->pitch);
        else
            transfer_function<double>(ctx, static_cast<cx<double>*>(out), w, h, wave->channels, tfc, wave->pitch);
    });
}

int holo_propagate(holo_ctx* ctx, const void* in, void* out, int w, int h, int c, const holo_wave* wave, double z,
                   const holo_prop_options* prop, int dtype) {
    return guarded([&] {
        require(ctx && in && out && wave, HOLO_ERR_USAGE, "null argument");
        check_dtype(dtype);
        if (w != wave->nx || h != wave->ny || c != wave->channels)
            config_error("propagate: field does not match the configured grid");  // propagation.cpp:94-95
        const holo_prop_options po = prop ? *prop : holo_prop_options{0, 0};
        if (dtype == HOLO_F32)
            op_propagate<float>(ctx, static_cast<const cx<float>*>(in), static_cast<cx<float>*>(out), w, h, c, *wave, z,
                                po);
        else
            op_propagate<double>(ctx, static_cast<const cx<double>*>(in), static_cast<cx<double>*>(out), w, h, c,
                                 *wave, z, po);
    });
}

int holo_forward_record(holo_ctx* ctx, const void* layers, int num_layers, void* hologram, const holo_wave* wave,
                        const holo_prop_options* prop, int dtype) {
    return guarded([&] {
        require(ctx && layers && hologram && wave, HOLO_ERR_USAGE, "null argument");
        check_dtype(dtype);
        const holo_prop_options po = prop ? *prop : holo_prop_options{0, 0};
        if (dtype == HOLO_F32)
            op_forward_record<float>(ctx, static_cast<const cx<float>*>(layers), num_layers,
                                     static_cast<cx<float>*>(hologram), *wave, po);
        else
            op_forward_record<double>(ctx, static_cast<const cx<double>*>(layers), num_layers,
                                      static_cast<cx<double>*>(hologram), *wave, po);
    });
}

int holo_inverse_propagate(holo_ctx* ctx, const void* hologram, void* replayed, const holo_wave* wave,
                           const holo_prop_options* prop, int dtype) {
    return guarded([&] {
        require(ctx && hologram && replayed && wave, HOLO_ERR_USAGE, "null argument");
        check_dtype(dtype);
        const holo_prop_options po = prop ? *prop : holo_prop_options{0, 0};
        if (dtype == HOLO_F32)
            op_inverse_propagate<float>(ctx, static_cast<const cx<float>*>(hologram), static_cast<cx<float>*>(replayed),
                                        *wave, po);
        else
            op_inverse_propagate<double>(ctx, static_cast<const cx<double>*>(hologram),
                                         static_cast<cx<double>*>(replayed), *wave, po);
    });
}

int holo_intensity_widened(holo_ctx* ctx, const void* field, double* out, size_t samples) {
    return guarded([&] {
        require(ctx && field && out, HOLO_ERR_USAGE, "null argument");
        if (samples == 0) return;
        const unsigned blocks = static_cast<unsigned>(std::min<size_t>((samples + 255) / 256, 16 * 148));
        k_intensity_widened<<<blocks, 256, 0, ctx->stream>>>(static_cast<const cx<float>*>(field), out, samples);
        HC_LAUNCHED(ctx);
    });
}

int holo_intensity(holo_ctx* ctx, const void* field, void* out, size_t samples, int dtype) {
    return guarded([&] {
        require(ctx && field && out, HOLO_ERR_USAGE, "null argument");
        check_dtype(dtype);
        if (samples == 0) return;
        if (dtype == HOLO_F32)
            intensity<float>(ctx, static_cast<const cx<float>*>(field), static_cast<float*>(out), samples);
        else
            intensity<double>(ctx, static_cast<const cx<double>*>(field), static_cast<double*>(out), samples);
    });
}

}  // extern "C"

// ---------------------------------------------------------------- training step

struct holo_optim {
    int device = 0;
    size_t n = 0;
    int planes = 0;
    bool sized = false;
    double* mom[7][4] = {};  // per group: m, v, n, prev_grad (OptimState::Moments)
    long long step = 0, skipped = 0;
};

namespace {

holo_loss_options loss_defaults(const holo_loss_options* o) {
    return o ? *o : holo_loss_options{0.005, 1e-4, 0};  // pipeline.hpp:26-28
}

// the loss terms of total_loss (pipeline.cpp:43-62) on device f64 stacks
void loss_terms(holo_ctx* ctx, const double* I, const double* G, const double* masks, int L, int C, int H, int W,
                const holo_loss_options& lo, bool with_ssim, double* grad, holo_loss_breakdown* out,
                double* psnr) {
    double* d_out = buf<double>(ctx, "loss_out", 1 + 2 * static_cast<size_t>(L));
    losses_gpu(ctx, I, G, masks, L, C, H, W, lo.use_plain_mse != 0, with_ssim, lo.lambda_ssim, grad, d_out);
    std::vector<double> h(1 + 2 * static_cast<size_t>(L));
    HC_CUDA(cudaMemcpyAsync(h.data(), d_out, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, ctx->stream));
    HC_CUDA(cudaStreamSynchronize(ctx->stream));
    out->recon = h[0];
    const double scale = lo.lambda_ssim / static_cast<double>(L);  // losses.cpp:98-104
    double ss = 0.0;
    for (int l = 0; l < L; ++l) ss += scale * (1.0 - h[1 + l]);
    out->ssim = ss;
    double acc = 0.0;
    for (int l = 0; l < L; ++l) {
        const double mse = h[1 + L + l];  // losses.cpp:129-131
        const double p = mse <= 0.0 ? 99.0 : std::min(99.0, 10.0 * std::log10(1.0 / mse));
        if (psnr) psnr[l] = p;
        acc += p;
    }
    out->psnr_mean = acc / static_cast<double>(L);
    out->opacity = 0.0;
    out->total = out->recon + out->ssim;
}

double cosine_lr(double base, double floor, long long t, long long total) {  // optimizer.cpp:7-11
    if (total <= 0 || t >= total) return floor;
    const double phase = 3.14159265358979323846 * static_cast<double>(t) / static_cast<double>(total);
    return floor + 0.5 * (base - floor) * (1.0 + std::cos(phase));
}

// the scene arrays the next render reads, ordered after any upload into them
holo_ctx::SceneSet& resident_scene(holo_ctx* ctx) {
    const int k = ctx->scene_cur;
    if (ctx->scene_wait[k]) {
        HC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_scene_ready[k], 0));
        ctx->scene_wait[k] = false;
    }
    return ctx->scene_sets[k];
}

}  // namespace

extern "C" {

int holo_losses(holo_ctx* ctx, const double* intensities, const double* targets, const double* masks, int L, int C,
                int H, int W, const holo_loss_options* opt, holo_loss_breakdown* out, double* psnr, double* grad) {
    return guarded([&] {
        require(ctx && intensities && targets && out, HOLO_ERR_USAGE, "null argument");
        require(L >= 1 && C >= 1 && H >= 1 && W >= 1, HOLO_ERR_CONFIG, "focal stack shape must be positive");
        const holo_loss_options lo = loss_defaults(opt);
        require(lo.use_plain_mse || masks, HOLO_ERR_USAGE, "masks are required unless use_plain_mse");
        HC_CUDA(cudaSetDevice(ctx->device));
        loss_terms(ctx, intensities, targets, masks, L, C, H, W, lo, lo.lambda_ssim != 0.0, grad, out, psnr);
    });
}

int holo_total_loss(holo_ctx* ctx, const holo_camera* cam, const holo_wave* wave, const holo_raster_settings* settings,
                    const holo_prop_options* prop, const holo_loss_options* opt, const double* targets,
                    const double* masks, holo_loss_breakdown* out, double* psnr, holo_scene_grads* grads) {
    return guarded([&] {
        require(ctx && cam && wave && settings && targets && out, HOLO_ERR_USAGE, "null argument");
        const holo_loss_options lo = loss_defaults(opt);
        require(lo.use_plain_mse || masks, HOLO_ERR_USAGE, "masks are required unless use_plain_mse");
        HC_CUDA(cudaSetDevice(ctx->device));
        validate_wave(*wave);
        const holo_prop_options po = prop ? *prop : holo_prop_options{0, 0};
        const int W = wave->nx, H = wave->ny, C = wave->channels, L = wave->num_planes;
        const size_t n = static_cast<size_t>(L) * C * H * W;
        render_full(ctx, *cam, *wave, *settings, po, HOLO_OUT_REPLAYED | HOLO_OUT_AUX, nullptr);
        // the intensities in f64 of the replayed fields (as intensity() of the
        // widened replay, so equal to what pipeline_forward's caller sees)
        const cx<float>* rep = static_cast<const cx<float>*>(ctx->buffer(out_name("replayed", ctx->out_sel), 1));
        double* i64 = buf<double>(ctx, "loss_I", n);
        replay_intensity_f64(ctx, rep, i64, n);
        double* gi = grads ? buf<double>(ctx, "loss_gI", n) : nullptr;
        loss_terms(ctx, i64, targets, masks, L, C, H, W, lo, true, gi, out, psnr);
        if (grads) pipeline_backward(ctx, *cam, *wave, *settings, po, nullptr, *grads, nullptr, nullptr, gi);
        // opacity decay (pipeline.cpp:47-52, 82-88) on the rendered scene
        const double* opac = ctx->scene_sets[ctx->f_scene_set].a[4];
        out->opacity = opacity_term(ctx, opac, ctx->n, lo.lambda_opacity, grads ? grads->opacity_logits : nullptr);
        out->total = out->recon + out->ssim + out->opacity;
    });
}

int holo_ssim(holo_ctx* ctx, const double* x, const double* y, int L, int C, int H, int W, double* mean_ssim,
              double* grad) {
    return guarded([&] {
        require(ctx && x && y && mean_ssim, HOLO_ERR_USAGE, "null argument");
        require(L >= 1 && C >= 1 && H >= 1 && W >= 1, HOLO_ERR_CONFIG, "image shape must be positive");
        HC_CUDA(cudaSetDevice(ctx->device));
        const size_t n = static_cast<size_t>(L) * C * H * W;
        if (grad) HC_CUDA(cudaMemsetAsync(grad, 0, sizeof(double) * n, ctx->stream));
        double* d_mean = buf<double>(ctx, "ssim_mean_out", static_cast<size_t>(L));
        ssim_gpu(ctx, x, y, L, C, H, W, -1.0, grad, d_mean);  // grad = 0 - (-1) g = g exactly
        HC_CUDA(cudaMemcpyAsync(mean_ssim, d_mean, sizeof(double) * L, cudaMemcpyDeviceToHost, ctx->stream));
        HC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int holo_plane_masks(holo_ctx* ctx, double* masks) {
    return guarded([&] {
        require(ctx && masks, HOLO_ERR_USAGE, "null argument");
        require(ctx->f_L > 0 && ctx->f_C > 0 && (ctx->f_outputs & HOLO_OUT_LAYERS), HOLO_ERR_USAGE,
                "plane masks need a frame rendered with HOLO_OUT_LAYERS");
        require(ctx->f_plane_begin == 0 && ctx->f_plane_end == ctx->f_L, HOLO_ERR_USAGE,
                "plane masks need every plane of the frame");
        HC_CUDA(cudaSetDevice(ctx->device));
        const size_t P = static_cast<size_t>(ctx->f_W) * ctx->f_H;
        const auto* layers = static_cast<const cx<float>*>(ctx->buffer("layers", 1));
        plane_masks(ctx, layers, ctx->f_L, ctx->f_C, P, masks);
    });
}

int holo_adaptive_update(holo_ctx* ctx, double* params, const double* grads, double* m, double* v, double* n,
                         double* prev_grad, size_t count, double lr, long long step,
                         const holo_optimizer_config* cfg) {
    return guarded([&] {
        require(ctx && cfg, HOLO_ERR_USAGE, "null argument");
        require(count == 0 || (params && grads && m && v && n && prev_grad), HOLO_ERR_USAGE, "null array");
        require(step >= 1, HOLO_ERR_USAGE, "step counts from 1");
        HC_CUDA(cudaSetDevice(ctx->device));
        adaptive_update(ctx, params, grads, m, v, n, prev_grad, count, lr, step, cfg->beta1, cfg->beta2, cfg->beta3,
                        cfg->eps, cfg->use_adam != 0);
    });
}

int holo_optim_create(holo_ctx* ctx, holo_optim** out) {
    return guarded([&] {
        require(ctx && out, HOLO_ERR_USAGE, "null argument");
        *out = new holo_optim();
        (*out)->device = ctx->device;
    });
}

int holo_optim_destroy(holo_optim* st) {
    if (!st) return HOLO_OK;
    cudaSetDevice(st->device);
    for (auto& g : st->mom)
        for (double* p : g) cudaFree(p);
    delete st;
    return HOLO_OK;
}

int holo_optim_counts(const holo_optim* st, long long* step, long long* skipped) {
    return guarded([&] {
        require(st, HOLO_ERR_USAGE, "null argument");
        if (step) *step = st->step;
        if (skipped) *skipped = st->skipped;
    });
}

int holo_optim_step(holo_ctx* ctx, holo_optim* st, const holo_scene_grads* grads, const holo_optimizer_config* cfg,
                    int* applied) {
    return guarded([&] {
        require(ctx && st && grads && cfg, HOLO_ERR_USAGE, "null argument");
        require(st->device == ctx->device, HOLO_ERR_USAGE, "optimizer state belongs to another device");
        HC_CUDA(cudaSetDevice(ctx->device));
        if (applied) *applied = 0;
        const size_t N = ctx->n;
        const int L = ctx->scene_planes;
        const size_t count[7] = {3 * N, 4 * N, 3 * N, 3 * N, N, 3 * N, N * static_cast<size_t>(L)};
        const double* g[7] = {grads->positions, grads->rotations, grads->log_scales, grads->amplitudes,
                              grads->opacity_logits, grads->phases, grads->plane_logits};
        for (int k = 0; k < 7; ++k)
            require(g[k] || count[k] == 0, HOLO_ERR_USAGE, "optimizer: every gradient group is required");
        if (!st->sized) {  // OptimState::resize_like (optimizer.cpp:41-49)
            for (int k = 0; k < 7; ++k)
                for (int j = 0; j < 4; ++j) {
                    HC_CUDA(cudaMalloc(&st->mom[k][j], sizeof(double) * (count[k] ? count[k] : 1)));
                    HC_CUDA(cudaMemsetAsync(st->mom[k][j], 0, sizeof(double) * (count[k] ? count[k] : 1), ctx->stream));
                }
            st->n = N;
            st->planes = L;
            st->sized = true;
        }
        require(st->n == N && st->planes == L, HOLO_ERR_CONFIG, "optimizer: moment buffers do not match the scene");
        holo_ctx::SceneSet& set = resident_scene(ctx);
        if (!grads_finite(ctx, g, count, 7)) {  // optimizer.cpp:110-115
            ++st->skipped;
            return;
        }
        const long long t = st->step;  // 0-based schedule position
        ++st->step;
        const double lr[7] = {cosine_lr(cfg->lr_positions, cfg->lr_floor, t, cfg->schedule_total),
                              cfg->lr_rotations,
                              cfg->lr_log_scales,
                              cfg->lr_amplitudes,
                              cfg->lr_opacities,
                              cfg->lr_phases,
                              cosine_lr(cfg->lr_plane_logits, cfg->lr_floor, t, cfg->schedule_total)};
        for (int k = 0; k < 7; ++k)
            adaptive_update(ctx, set.a[k], g[k], st->mom[k][0], st->mom[k][1], st->mom[k][2], st->mom[k][3], count[k],
                            lr[k], st->step, cfg->beta1, cfg->beta2, cfg->beta3, cfg->eps, cfg->use_adam != 0);
        renormalize_scene(ctx, set.a[1], set.a[3], N);  // scene.cpp:34-47
        if (applied) *applied = 1;
    });
}

int holo_scene_download(holo_ctx* ctx, const holo_scene_arrays* host) {
    return guarded([&] {
        require(ctx && host, HOLO_ERR_USAGE, "null argument");
        require(host->n == ctx->n && host->num_planes == ctx->scene_planes, HOLO_ERR_USAGE,
                "scene download: n / num_planes differ from the resident scene");
        HC_CUDA(cudaSetDevice(ctx->device));
        const size_t N = ctx->n;
        const size_t count[7] = {3 * N, 4 * N, 3 * N, 3 * N, N, 3 * N, N * static_cast<size_t>(ctx->scene_planes)};
        const double* dst[7] = {host->positions, host->rotations, host->log_scales, host->amplitudes,
                                host->opacity_logits, host->phases, host->plane_logits};
        holo_ctx::SceneSet& set = resident_scene(ctx);
        for (int k = 0; k < 7; ++k)
            if (count[k]) {
                require(dst[k] != nullptr, HOLO_ERR_USAGE, "scene download: null array");
                HC_CUDA(cudaMemcpyAsync(const_cast<double*>(dst[k]), set.a[k], sizeof(double) * count[k],
                                        cudaMemcpyDeviceToHost, ctx->stream));
            }
        HC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"

// ---------------------------------------------------------------- phase-only conversion

namespace {

// phase_only.cpp:22-101 on device f64 fields.  The reference stack is replayed
// once (MatchTargets); each evaluation replays e^{j theta} to every plane from one
// spectrum, and the gradient pulls all planes back through one summed spectrum
// (the sum of the per-plane propagate(+z) calls, by linearity, crop included).
struct PhaseProblem {
    holo_wave wave{};
    holo_prop_options po{};
    int w = 0, h = 0, C = 0, L = 0, pw = 0, ph = 0, oy = 0;
    bool pad = false;
    size_t n = 0, gn = 0;
    std::vector<double> z;
    cx<double>* tf = nullptr;   // target fields [L][C][h][w]
    double* timg = nullptr;     // target intensities
    const TfChan* tfc = nullptr;
    cx<double>* tab = nullptr;  // H_{Z_l} on the (padded) grid [L][C][ph][pw], computed once
    const int* planes = nullptr;  // 0..L-1
    const int* none = nullptr;    // -1
};

PhaseProblem phase_problem(holo_ctx* ctx, const cx<double>* P, const holo_wave& wave, const holo_prop_options& po) {
    validate_wave(wave);  // cfg.validate (phase_only.cpp:23)
    PhaseProblem p;
    p.wave = wave;
    p.po = po;
    p.w = wave.nx;
    p.h = wave.ny;
    p.C = wave.channels;
    p.L = wave.num_planes;
    p.pad = po.pad2x != 0;
    p.pw = p.pad ? 2 * p.w : p.w;
    p.ph = p.pad ? 2 * p.h : p.h;
    p.oy = (p.ph - p.h) / 2;  // pad_center (propagation.cpp:64-72)
    p.n = static_cast<size_t>(p.C) * p.w * p.h;
    p.gn = static_cast<size_t>(p.C) * p.pw * p.ph;
    p.z = plane_positions(wave);
    if (p.w < 11 || p.h < 11) config_error("ssim needs images at least 11 pixels in each dimension");
    if (!all_finite_c128(ctx, P, p.n)) throw Error(HOLO_ERR_NUMERIC, "hologram contains non-finite samples");
    p.tf = buf<cx<double>>(ctx, "po_tf", p.n * p.L);
    p.timg = buf<double>(ctx, "po_timg", p.n * p.L);
    op_inverse_propagate<double>(ctx, P, p.tf, wave, po);  // replay_targets (phase_only.cpp:31-38)
    intensity<double>(ctx, p.tf, p.timg, p.n * p.L);
    // the planes' transfer functions on the propagation grid, once for the whole
    // conversion (the same values the column passes would evaluate per element)
    p.tfc = upload_tf(ctx, "po_tfc", wave, p.z, p.pw, p.ph, po.local_band_limit);
    p.tab = buf<cx<double>>(ctx, "po_tftab", p.gn * p.L);
    for (int l = 0; l < p.L; ++l)
        transfer_function<double>(ctx, p.tab + p.gn * l, p.pw, p.ph, p.C, p.tfc + l * p.C, wave.pitch);
    std::vector<int> pl(p.L);
    for (int l = 0; l < p.L; ++l) pl[l] = l;
    int* d_pl = buf<int>(ctx, "po_planes", p.L);
    upload_small(ctx, d_pl, pl.data(), sizeof(int) * p.L);
    int* d_none = buf<int>(ctx, "po_none", 1);
    const int m1 = -1;
    upload_small(ctx, d_none, &m1, sizeof(int));
    p.planes = d_pl;
    p.none = d_none;
    return p;
}

// row FFTs of the rows [oy, oy + h) of each of `fields` (padded) grids: the other
// rows are zero on input (forward) or never read (inverse)
void crop_rows_fft(holo_ctx* ctx, const PhaseProblem& p, cx<double>* f, int fields, int dir) {
    const double s = dir > 0 ? 1.0 / (static_cast<double>(p.pw) * p.ph) : 1.0;
    for (int k = 0; k < fields; ++k) {
        cx<double>* r = f + static_cast<size_t>(k) * p.ph * p.pw + static_cast<size_t>(p.oy) * p.pw;
        rows_fft<double>(ctx, r, r, p.pw, p.h, dir, s);
    }
}

// eval_loss (phase_only.cpp:48-101); grad (device, optional) = d loss / d theta
double phase_eval(holo_ctx* ctx, const PhaseProblem& p, const double* theta, double lambda_ssim, double* grad) {
    const int w = p.w, h = p.h, C = p.C, L = p.L;
    cx<double>* cand = buf<cx<double>>(ctx, "po_cand", p.gn);
    cx<double>* rep = buf<cx<double>>(ctx, "po_rep", p.gn * L);
    double* img = buf<double>(ctx, "po_img", p.n * L);
    double* sums = buf<double>(ctx, "po_sums", 2 * static_cast<size_t>(L));
    const ColOpts<double> band{p.tab, p.oy, p.oy + h};
    // e^{j theta} -> spectrum (row pass pruned to the field's rows)
    phase_field(ctx, theta, cand, w, h, C, p.pad);
    crop_rows_fft(ctx, p, cand, C, -1);
    cols_fft<double>(ctx, cand, cand, p.pw, p.ph, C, -1, 1.0);
    // replays: column IFFT with H_{-Z_l}, the cropped rows only, then their row IFFT
    col_replay<double>(ctx, cand, rep, p.pw, p.ph, C, L, p.planes, p.tfc, p.wave.pitch, band);
    crop_rows_fft(ctx, p, rep, L * C, +1);
    phase_match(ctx, rep, p.tf, w, h, C, L, p.pad, img, sums);
    double* gi = nullptr;
    if (grad) {
        gi = buf<double>(ctx, "po_gi", p.n * L);
        HC_CUDA(cudaMemsetAsync(gi, 0, sizeof(double) * p.n * L, ctx->stream));
    }
    if (lambda_ssim != 0.0) ssim_gpu(ctx, img, p.timg, L, C, h, w, lambda_ssim / L, gi, sums + L);
    std::vector<double> hs(2 * static_cast<size_t>(L), 1.0);
    HC_CUDA(cudaMemcpyAsync(hs.data(), sums, sizeof(double) * (lambda_ssim != 0.0 ? 2 * L : L),
                            cudaMemcpyDeviceToHost, ctx->stream));
    const double inv_lm = 1.0 / (static_cast<double>(L) * static_cast<double>(p.n));
    if (grad) {
        // seed over the cropped rows, one summed spectrum sum_l H_{Z_l} FFT(gv_l),
        // one inverse transform (again pruned to the cropped rows)
        phase_seed(ctx, rep, p.tf, gi, w, h, C, L, p.pad, inv_lm);
        crop_rows_fft(ctx, p, rep, L * C, -1);
        col_spectrum<double>(ctx, rep, cand, p.pw, p.ph, C, L, p.tfc, p.wave.pitch, band);
        cx<double>* acc = buf<cx<double>>(ctx, "po_acc", p.gn);
        col_replay<double>(ctx, cand, acc, p.pw, p.ph, C, 1, p.none, p.tfc, p.wave.pitch, band);
        crop_rows_fft(ctx, p, acc, C, +1);
        phase_grad(ctx, acc, theta, grad, w, h, C, p.pad);
    }
    HC_CUDA(cudaStreamSynchronize(ctx->stream));
    double field_term = 0.0, ssim_term = 0.0;
    for (int l = 0; l < L; ++l) field_term += hs[l] * inv_lm;
    const double scale = lambda_ssim / static_cast<double>(L);  // losses.cpp:98-104
    for (int l = 0; l < L; ++l) ssim_term += scale * (1.0 - hs[L + l]);
    return field_term + ssim_term;
}

}  // namespace

extern "C" {

int holo_phase_only_loss(holo_ctx* ctx, const void* P, const double* theta, const holo_wave* wave,
                         const holo_phase_options* opt, double* loss, double* grad) {
    return guarded([&] {
        require(ctx && P && theta && wave && opt && loss, HOLO_ERR_USAGE, "null argument");
        HC_CUDA(cudaSetDevice(ctx->device));
        const PhaseProblem p = phase_problem(ctx, static_cast<const cx<double>*>(P), *wave, opt->prop);
        *loss = phase_eval(ctx, p, theta, opt->lambda_ssim, grad);
    });
}

int holo_convert_phase_only(holo_ctx* ctx, const void* P, const holo_wave* wave, int iters, double lr,
                            const holo_phase_options* opt, const double* theta0, double* phase_out, double* trace) {
    return guarded([&] {
        require(ctx && P && wave && opt && phase_out && trace, HOLO_ERR_USAGE, "null argument");
        HC_CUDA(cudaSetDevice(ctx->device));
        const cx<double>* Pd = static_cast<const cx<double>*>(P);
        validate_wave(*wave);
        if (iters < 0) config_error("iteration count must be non-negative");  // phase_only.cpp:116-117
        if (!(lr > 0.0)) config_error("step size must be positive");
        const PhaseProblem p = phase_problem(ctx, Pd, *wave, opt->prop);
        const size_t N = p.n;
        double* theta = buf<double>(ctx, "po_theta", N);
        if (theta0)
            HC_CUDA(cudaMemcpyAsync(theta, theta0, sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
        else
            phase_arg(ctx, Pd, theta, N);  // theta = arg(P) (phase_only.cpp:124-126)
        double* g = buf<double>(ctx, "po_g", N);
        double loss = phase_eval(ctx, p, theta, opt->lambda_ssim, iters > 0 ? g : nullptr);
        trace[0] = loss;
        if (iters == 0) {
            HC_CUDA(cudaMemcpyAsync(phase_out, theta, sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
            HC_CUDA(cudaStreamSynchronize(ctx->stream));
            return;
        }
        // OptimizerConfig defaults with use_adam from the options (phase_only.cpp:138-141)
        const double b1 = 0.9, b2 = 0.99, b3 = 0.99, eps = 1e-8;
        double* mom = buf<double>(ctx, "po_mom", 4 * N);
        HC_CUDA(cudaMemsetAsync(mom, 0, sizeof(double) * 4 * N, ctx->stream));
        double* best = buf<double>(ctx, "po_best", N);
        HC_CUDA(cudaMemcpyAsync(best, theta, sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
        double best_loss = loss, prev = loss, step_lr = lr;
        for (int it = 1; it <= iters; ++it) {
            adaptive_update(ctx, theta, g, mom, mom + N, mom + 2 * N, mom + 3 * N, N, step_lr, it, b1, b2, b3, eps,
                            opt->use_adam != 0);
            loss = phase_eval(ctx, p, theta, opt->lambda_ssim, g);
            trace[it] = loss;
            if (loss < best_loss) {
                best_loss = loss;
                HC_CUDA(cudaMemcpyAsync(best, theta, sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
            }
            if (loss > prev) {  // backtrack: halve the step, restart from the best iterate
                step_lr *= 0.5;
                HC_CUDA(cudaMemcpyAsync(theta, best, sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
                loss = phase_eval(ctx, p, theta, opt->lambda_ssim, g);
            }
            prev = loss;
        }
        HC_CUDA(cudaMemcpyAsync(phase_out, best, sizeof(double) * N, cudaMemcpyDeviceToDevice, ctx->stream));
        HC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
