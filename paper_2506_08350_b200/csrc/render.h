// Frame-level entry points shared by capi.cu and the group renderer (group.cu).
// Internal to libholo_cuda.
#pragma once

#include <new>

#include "kernels.cuh"

namespace holo_cuda {

// holo_last_error() of this thread
void set_last_error(const char* msg);

// run f, mapping exceptions to a status code and holo_last_error()
template <class F>
int guarded_call(F&& f) {
    try {
        f();
        return HOLO_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return HOLO_ERR_OOM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return HOLO_ERR_NUMERIC;
    }
}

inline void require(bool ok, int code, const char* msg) {
    if (!ok) throw Error(code, msg);
}

// holo_render's body (pipeline_forward, pipeline.cpp:20-29) on one context
void render_whole(holo_ctx* ctx, const holo_camera& cam, const holo_wave& wave, const holo_raster_settings& st,
                  const holo_prop_options& po, unsigned outputs, holo_frame_info* info);
// create the per-channel events of a plane-sharded frame (idempotent)
void chan_events(holo_ctx* ctx);
// planes [pb, pe): raster, column FFT, then the partial spectrum channel by
// channel into spec; ctx->ev_chan_ready[c] recorded after channel c
void shard_front(holo_ctx* ctx, const holo_camera& cam, const holo_wave& wave, const holo_raster_settings& st,
                 const holo_prop_options& po, int pb, int pe, unsigned outputs, cx<float>* spec,
                 holo_frame_info* info);
// from the summed spectrum: channel c waits for ctx->ev_chan_done[c], then the
// replays of planes [pb, pe) and the hologram channels in holo_mask
void shard_back(holo_ctx* ctx, const holo_wave& wave, const holo_prop_options& po, int pb, int pe,
                const cx<float>* spec, unsigned outputs, unsigned holo_mask);
// destination of the current frame's hologram ([C][H][W] complex64)
cx<float>* frame_hologram(holo_ctx* ctx, int C, size_t P);
// keep the Gaussians of planes [pb, pe) (hard assignment), in order
void scene_restrict_planes(holo_ctx* ctx, int pb, int pe);
// copy from's current scene into to (same device)
void scene_replicate(holo_ctx* from, holo_ctx* to);

}  // namespace holo_cuda
