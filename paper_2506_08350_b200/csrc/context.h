// holo_ctx: one CUDA stream, grow-only device scratch, the resident scene and the
// last frame's outputs.  Internal to libholo_cuda.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "fft.cuh"

namespace holo_cuda {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    size_t guard_at = 0;  // guard mode: offset of the guard band (the requested size)
};

// Guard mode (HOLO_GUARD=1 at context creation, or holo_ctx_set_guard): every
// scratch buffer is allocated at its exact requested size followed by a band of
// kGuardBytes set to kGuardByte; holo_ctx_check_guards (and every reallocation)
// verifies the bands -- an out-of-bounds write past any buffer is reported by
// name.  The substitute for compute-sanitizer memcheck, which this pool disables.
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kGuardByte = 0xA5;

// Per-(plane, channel) transfer-function constants, see tf_value() in kernels.cuh.
struct TfChan {
    double inv_l2;      // 1 / lambda^2
    double two_pi_z;    // 2 pi z (f64, as propagation.cpp:51)
    double fx_lim, fy_lim;
    float inv_l;        // 1 / lambda
    float two_pi_z_f;   // 2 pi z
    float phase0;       // (2 pi z / lambda) mod 2 pi
    int local;          // local band limit active (opt && z != 0)
    // step to the next plane (the row pass's plane recurrence, render_static.cu):
    // (2 pi dz / lambda) mod 2 pi and 2 pi dz, dz = z_{l+1} - z_l (f64, then fp32)
    float step_phase;
    float step_2piz;
};

constexpr int kNumStages = 8;

}  // namespace holo_cuda

struct holo_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    uint64_t launches = 0;

    // stage timing (CUDA events on the context stream)
    bool timing = false;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    double stage_ms[holo_cuda::kNumStages] = {};
    int stage_calls[holo_cuda::kNumStages] = {};

    std::map<std::string, holo_cuda::DevBuf> scratch;
    bool guard = false;
    // single-pass scans (binning.cu): epoch and ticket base of the next call, and
    // the tile capacity of the zero-initialised status words
    struct ScanState {
        unsigned epoch = 0, ticket = 0;
        int cap = 0;
    } scan;
    std::map<std::pair<int, int>, void*> twiddles;      // (n, sizeof(T)) -> exp(-2 pi i q/n)
    std::map<std::pair<int, uint64_t>, double*> freqs;  // (n, pitch bits) -> freq_at(i, n, pitch)
    std::map<std::string, void*> tables;                 // frame-invariant device tables (render_static.cu)
    std::map<const void*, std::vector<holo_cuda::TfChan>> tf_host;  // host copy of each uploaded TF table
    void* host_pinned = nullptr;
    size_t host_pinned_bytes = 0;

    // resident scene (device, f64 SoA), double-buffered: a host upload fills the set
    // the previous frame is not reading, on the copy-in stream, while that frame
    // renders; d_* point at the set the next render reads
    size_t n = 0;
    int scene_planes = 0;
    double* d_positions = nullptr;
    double* d_rotations = nullptr;
    double* d_log_scales = nullptr;
    double* d_amplitudes = nullptr;
    double* d_opacity = nullptr;
    double* d_phases = nullptr;
    double* d_plane_logits = nullptr;
    struct SceneSet {
        double* a[7] = {};  // positions, rotations, log_scales, amplitudes, opacity, phases, plane_logits
        size_t cap[7] = {};
    };
    SceneSet scene_sets[2];
    int scene_cur = 0;
    cudaStream_t copy_in = nullptr, copy_out = nullptr;  // non-blocking copy streams
    cudaEvent_t ev_scene_ready[2] = {};  // upload into set k complete (copy_in)
    cudaEvent_t ev_scene_free[2] = {};   // last reader of set k (preprocess) done (stream)
    bool scene_wait[2] = {};             // the next render must wait for ev_scene_ready[k]
    // the final outputs (hologram, replayed, intensity) alternate between two buffer
    // sets frame by frame, so a frame's last pass need not wait for the download of
    // the previous frame's outputs
    int out_sel = 0;                        // set written by the last render
    cudaEvent_t ev_out_src = nullptr;       // frame work enqueued before an async download
    cudaEvent_t ev_out_done[2] = {};        // async downloads from set k complete (copy_out)
    unsigned out_pending[2] = {};           // buffer ids (bit per HOLO_BUF_*) with downloads in flight, per set
    // caller-owned destinations of the final outputs (a multi-view group render
    // writes each view straight into its own buffers); null = the context's sets
    void* out_dest[3] = {};                 // hologram, replayed, intensities
    // per-channel events of a plane-sharded frame: partial spectrum of channel c
    // written (stream) / its sum over the plane group complete (comm stream)
    cudaEvent_t ev_chan_ready[HOLO_MAX_CHANNELS] = {};
    cudaEvent_t ev_chan_done[HOLO_MAX_CHANNELS] = {};

    // last frame
    int f_L = 0, f_C = 0, f_W = 0, f_H = 0, f_tiles = 0;
    int f_tiles_x = 0, f_tiles_y = 0;
    long long f_buckets = 0;
    uint64_t f_E = 0;
    unsigned f_num_valid = 0, f_max_bucket = 0;
    unsigned f_outputs = 0;
    int f_plane_begin = 0, f_plane_end = 0;
    holo_camera f_cam{};            // camera and settings of the last render (the backward
    holo_raster_settings f_st{};    // must be called with the same ones)
    int f_scene_set = 0;            // scene set the last render read

    // asynchronous frames (holo_ctx_set_async): no host round trip inside a frame;
    // the entry buffers hold e_cap entries and each frame's status words
    // (flags, num_valid, max bucket, -, E) land in a pinned ring, consumed in order
    bool async = false;
    size_t e_cap = 0;
    unsigned f_cap = 0;               // entry-buffer capacity of the last frame
    static constexpr int kStatusSlots = 8;
    static constexpr int kStatusWords = 8;
    unsigned* host_status = nullptr;  // pinned, (kStatusSlots + 1) x kStatusWords; the last slot serves synchronous frames
    cudaEvent_t status_events[kStatusSlots] = {};
    int status_order[kStatusSlots] = {};  // pending slots, oldest first
    int status_pending_n = 0, status_next = 0;
    unsigned sticky_flags = 0;        // validation / overflow flags of consumed asynchronous frames

    // stage-timing event pairs awaiting resolution, and a pool of spare events
    struct Timed {
        int stage;
        cudaEvent_t a, b;
    };
    std::vector<Timed> pending;
    std::vector<cudaEvent_t> event_pool;
    // pinned ring for small asynchronous table uploads
    static constexpr int kRingSlots = 64;
    static constexpr size_t kRingSlotBytes = 64 * 1024;
    std::map<const void*, std::vector<unsigned char>> small_cache;  // last table uploaded per device buffer
    unsigned char* ring = nullptr;
    cudaEvent_t ring_ev[kRingSlots] = {};
    bool ring_used[kRingSlots] = {};
    int ring_next = 0;

    void note_launch() { ++launches; }
    void* buffer(const std::string& name, size_t bytes);
    void* pinned(size_t bytes);
    template <class T>
    const holo_cuda::cx<T>* twiddle(int n);
    const double* freq(int n, double pitch);
    void stage_begin();
    void stage_end(int stage);
};
