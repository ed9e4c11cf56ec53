// Multi-GPU groups: plane sharding, view sharding and the planes x views mesh
// (include/holo_cuda.h, SURVEY.md 8(b) holo_group_*, 8(e)).
//
// One frame is pipeline_forward (pipeline.cpp:20-29).  Its forward recording is a
// sum over planes (propagation.cpp:103-114), linear in the layers, so a plane group
// splits the planes, each rank forms its partial spectrum S_g channel by channel
// (shard_front), the group sums channel c while the row pass of channel c + 1 runs,
// and each rank replays its own planes and forms the hologram channels it owns
// (shard_back).  Views are independent frames of one resident scene (the views
// train iterates, trainer.cpp:118-133): no per-frame collective.  world =
// view_groups x plane_split; the spectrum sum runs inside each plane group.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, reusing an already loaded
// copy such as torch's), so the library carries no link-time NCCL dependency and
// the single-GPU entry points work where NCCL is absent.
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only; the symbols come from dlsym

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "render.h"

using namespace holo_cuda;

namespace {

// ---------------------------------------------------------------- NCCL at run time

struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommInitAll) CommInitAll = nullptr;
    decltype(&ncclCommSplit) CommSplit = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    std::string error;
};

NcclApi load_nccl() {
    NcclApi api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        const char* e = dlerror();
        api.error = std::string("NCCL not found: ") + (e ? e : "dlopen failed");
        return api;
    }
#define HG_SYM(name)                                                              \
    api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name));      \
    if (!api.name) {                                                              \
        api.error = "NCCL lacks nccl" #name;                                      \
        return api;                                                               \
    }
    HG_SYM(GetUniqueId)
    HG_SYM(CommInitRank)
    HG_SYM(CommInitAll)
    HG_SYM(CommSplit)
    HG_SYM(CommDestroy)
    HG_SYM(AllReduce)
    HG_SYM(GroupStart)
    HG_SYM(GroupEnd)
    HG_SYM(GetErrorString)
#undef HG_SYM
    return api;
}

const NcclApi& nccl() {
    static const NcclApi api = load_nccl();
    if (!api.error.empty()) throw Error(HOLO_ERR_NCCL, api.error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(HOLO_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// ---------------------------------------------------------------- mesh arithmetic

std::pair<int, int> balanced_range(int n, int parts, int k) {
    const int base = n / parts, extra = n % parts;
    const int b = k * base + std::min(k, extra);
    return {b, b + base + (k < extra ? 1 : 0)};
}

holo_mesh layout(int world, int rank, int plane_split, int num_planes, int num_views, int channels) {
    if (world < 1 || rank < 0 || rank >= world)
        throw Error(HOLO_ERR_USAGE, "group: rank outside [0, world)");
    if (plane_split < 1 || world % plane_split != 0)
        throw Error(HOLO_ERR_USAGE, "group: plane_split must divide the world size");
    if (num_planes < 0 || num_views < 0 || channels < 0 || channels > HOLO_MAX_CHANNELS)
        throw Error(HOLO_ERR_USAGE, "group: negative plane / view / channel count");
    holo_mesh m{};
    m.world = world;
    m.rank = rank;
    m.plane_split = plane_split;
    m.view_groups = world / plane_split;
    m.plane_rank = rank % plane_split;
    m.view_group = rank / plane_split;
    const auto pr = balanced_range(num_planes, plane_split, m.plane_rank);
    m.plane_begin = pr.first;
    m.plane_end = pr.second;
    const auto vr = balanced_range(num_views, m.view_groups, m.view_group);
    m.view_begin = vr.first;
    m.view_end = vr.second;
    for (int c = 0; c < channels; ++c)
        if (c % plane_split == m.plane_rank) m.holo_channels |= 1u << c;
    return m;
}

}  // namespace

// ---------------------------------------------------------------- the group

struct holo_group {
    enum Transport { kNccl, kCallback };
    struct Lane {
        holo_ctx* ctx = nullptr;
        bool owned = false;
        cudaStream_t comm = nullptr;  // collectives of this lane's frames
        cudaEvent_t ev_holo = nullptr;
    };
    struct Local {
        int rank = 0;
        int device = 0;
        unsigned long long frames = 0;  // frames rendered: the lane of the next one rotates across calls
        ncclComm_t world_comm = nullptr;
        ncclComm_t plane_comm = nullptr;  // the plane group's (== world_comm when one group spans the world)
        std::vector<Lane> lanes;
    };
    int world = 1, plane_split = 1;
    Transport transport = kNccl;
    holo_allreduce_fn fn = nullptr;
    void* user = nullptr;
    std::vector<Local> locals;
};

namespace {

holo_group::Lane make_lane(holo_ctx* ctx, bool owned) {
    holo_group::Lane ln;
    ln.ctx = ctx;
    ln.owned = owned;
    HC_CUDA(cudaSetDevice(ctx->device));
    HC_CUDA(cudaStreamCreateWithFlags(&ln.comm, cudaStreamNonBlocking));
    HC_CUDA(cudaEventCreateWithFlags(&ln.ev_holo, cudaEventDisableTiming));
    chan_events(ctx);
    return ln;
}

void free_lane(holo_group::Lane& ln) {
    if (ln.ctx) {
        cudaSetDevice(ln.ctx->device);
        cudaStreamSynchronize(ln.comm);
    }
    if (ln.comm) cudaStreamDestroy(ln.comm);
    if (ln.ev_holo) cudaEventDestroy(ln.ev_holo);
    if (ln.owned && ln.ctx) holo_ctx_destroy(ln.ctx);
    ln = holo_group::Lane{};
}

// the plane communicators of several local ranks: ncclCommSplit inside one group call
void split_planes(holo_group* g) {
    if (g->plane_split == g->world) {  // one plane group (also a world of one)
        for (auto& l : g->locals) l.plane_comm = l.world_comm;
        return;
    }
    if (g->plane_split == 1) return;  // views only: no spectrum sums
    const NcclApi& n = nccl();
    nccl_check(n.GroupStart(), "ncclGroupStart");
    for (auto& l : g->locals) {
        HC_CUDA(cudaSetDevice(l.device));
        nccl_check(n.CommSplit(l.world_comm, l.rank / g->plane_split, l.rank % g->plane_split, &l.plane_comm, nullptr),
                   "ncclCommSplit");
    }
    nccl_check(n.GroupEnd(), "ncclGroupEnd");
}

// sum `count` floats at buf[i] over each local rank's plane group, on lane i's
// comm stream after `ready[i]`; `done[i]` recorded when the sum is complete
void plane_sum(holo_group* g, const std::vector<holo_group::Lane*>& lanes, const std::vector<int>& who,
               const std::vector<float*>& bufs, size_t count, const std::vector<cudaEvent_t>& ready,
               const std::vector<cudaEvent_t>& done) {
    for (size_t i = 0; i < lanes.size(); ++i) {
        HC_CUDA(cudaSetDevice(lanes[i]->ctx->device));
        HC_CUDA(cudaStreamWaitEvent(lanes[i]->comm, ready[i], 0));
    }
    if (g->transport == holo_group::kCallback) {
        for (size_t i = 0; i < lanes.size(); ++i) {
            const int rc = g->fn(g->user, bufs[i], count, lanes[i]->comm);
            if (rc != 0) throw Error(HOLO_ERR_NCCL, "group: all-reduce callback failed (" + std::to_string(rc) + ")");
        }
    } else if (g->locals[who[0]].plane_comm) {
        const NcclApi& n = nccl();
        nccl_check(n.GroupStart(), "ncclGroupStart");
        for (size_t i = 0; i < lanes.size(); ++i) {
            HC_CUDA(cudaSetDevice(lanes[i]->ctx->device));
            nccl_check(n.AllReduce(bufs[i], bufs[i], count, ncclFloat32, ncclSum, g->locals[who[i]].plane_comm,
                                   lanes[i]->comm),
                       "ncclAllReduce");
        }
        nccl_check(n.GroupEnd(), "ncclGroupEnd");
    }
    // plane groups of one (HOLO_GROUP_SHARDED_PATH): the partial spectrum is the sum
    for (size_t i = 0; i < lanes.size(); ++i) {
        HC_CUDA(cudaSetDevice(lanes[i]->ctx->device));
        HC_CUDA(cudaEventRecord(done[i], lanes[i]->comm));
    }
}

void check_group(const holo_group* g) { require(g != nullptr, HOLO_ERR_USAGE, "null group"); }

}  // namespace

extern "C" {

int holo_mesh_layout(int world, int rank, int plane_split, int num_planes, int num_views, int channels,
                     holo_mesh* out) {
    return guarded_call([&] {
        require(out != nullptr, HOLO_ERR_USAGE, "null argument");
        *out = layout(world, rank, plane_split, num_planes, num_views, channels);
    });
}

int holo_group_unique_id(unsigned char id[HOLO_GROUP_ID_BYTES]) {
    return guarded_call([&] {
        require(id != nullptr, HOLO_ERR_USAGE, "null argument");
        static_assert(sizeof(ncclUniqueId) == HOLO_GROUP_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId u;
        nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof u);
    });
}

int holo_group_init_rank(holo_ctx* ctx, const unsigned char id[HOLO_GROUP_ID_BYTES], int world, int rank,
                         int plane_split, holo_group** out) {
    return guarded_call([&] {
        require(ctx && id && out, HOLO_ERR_USAGE, "null argument");
        (void)layout(world, rank, plane_split, 0, 0, 0);
        auto* g = new holo_group();
        g->world = world;
        g->plane_split = plane_split;
        g->transport = holo_group::kNccl;
        holo_group::Local l;
        l.rank = rank;
        l.device = ctx->device;
        try {
            HC_CUDA(cudaSetDevice(ctx->device));
            ncclUniqueId u;
            std::memcpy(&u, id, sizeof u);
            nccl_check(nccl().CommInitRank(&l.world_comm, world, u, rank), "ncclCommInitRank");
            l.lanes.push_back(make_lane(ctx, false));
            g->locals.push_back(l);
            split_planes(g);
        } catch (...) {
            for (auto& ln : l.lanes) free_lane(ln);
            delete g;
            throw;
        }
        *out = g;
    });
}

int holo_group_init_callback(holo_ctx* ctx, int world, int rank, int plane_split, holo_allreduce_fn fn, void* user,
                             holo_group** out) {
    return guarded_call([&] {
        require(ctx && fn && out, HOLO_ERR_USAGE, "null argument");
        (void)layout(world, rank, plane_split, 0, 0, 0);
        auto* g = new holo_group();
        g->world = world;
        g->plane_split = plane_split;
        g->transport = holo_group::kCallback;
        g->fn = fn;
        g->user = user;
        holo_group::Local l;
        l.rank = rank;
        l.device = ctx->device;
        l.lanes.push_back(make_lane(ctx, false));
        g->locals.push_back(l);
        *out = g;
    });
}

int holo_group_create(const int* devices, int n, int plane_split, holo_group** out) {
    return guarded_call([&] {
        require(devices && out && n >= 1, HOLO_ERR_USAGE, "holo_group_create: need at least one device");
        (void)layout(n, 0, plane_split, 0, 0, 0);
        auto* g = new holo_group();
        g->world = n;
        g->plane_split = plane_split;
        try {
            std::vector<ncclComm_t> comms(n, nullptr);
            nccl_check(nccl().CommInitAll(comms.data(), n, devices), "ncclCommInitAll");
            for (int i = 0; i < n; ++i) {
                holo_group::Local l;
                l.rank = i;
                l.device = devices[i];
                l.world_comm = comms[i];
                holo_ctx* c = nullptr;
                if (holo_ctx_create(devices[i], &c) != HOLO_OK) throw Error(HOLO_ERR_CUDA, holo_last_error());
                l.lanes.push_back(make_lane(c, true));
                g->locals.push_back(l);
            }
            split_planes(g);
        } catch (...) {
            holo_group_destroy(g);
            throw;
        }
        *out = g;
    });
}

int holo_group_destroy(holo_group* g) {
    return guarded_call([&] {
        if (!g) return;
        for (auto& l : g->locals) {
            for (auto& ln : l.lanes) free_lane(ln);
            if (g->transport == holo_group::kNccl) {
                const NcclApi& n = nccl();
                if (l.plane_comm && l.plane_comm != l.world_comm) n.CommDestroy(l.plane_comm);
                if (l.world_comm) n.CommDestroy(l.world_comm);
            }
        }
        delete g;
    });
}

int holo_group_local_count(const holo_group* g) { return g ? static_cast<int>(g->locals.size()) : 0; }

int holo_group_context(holo_group* g, int local, holo_ctx** ctx) {
    return guarded_call([&] {
        check_group(g);
        require(ctx && local >= 0 && local < static_cast<int>(g->locals.size()), HOLO_ERR_USAGE,
                "group: no such local rank");
        *ctx = g->locals[local].lanes[0].ctx;
    });
}

int holo_group_mesh(const holo_group* g, int local, int num_planes, int num_views, int channels, holo_mesh* out) {
    return guarded_call([&] {
        check_group(g);
        require(out && local >= 0 && local < static_cast<int>(g->locals.size()), HOLO_ERR_USAGE,
                "group: no such local rank");
        *out = layout(g->world, g->locals[local].rank, g->plane_split, num_planes, num_views, channels);
    });
}

int holo_group_set_lanes(holo_group* g, int lanes) {
    return guarded_call([&] {
        check_group(g);
        require(lanes >= 1 && lanes <= 8, HOLO_ERR_USAGE, "group: lanes must be in [1, 8]");
        for (auto& l : g->locals) {
            while (static_cast<int>(l.lanes.size()) > lanes) {
                free_lane(l.lanes.back());
                l.lanes.pop_back();
            }
            while (static_cast<int>(l.lanes.size()) < lanes) {
                holo_ctx* c = nullptr;
                if (holo_ctx_create(l.device, &c) != HOLO_OK) throw Error(HOLO_ERR_CUDA, holo_last_error());
                holo_ctx* primary = l.lanes[0].ctx;
                c->async = primary->async;
                c->e_cap = primary->e_cap;
                l.lanes.push_back(make_lane(c, true));
                if (primary->n > 0 || primary->scene_planes > 0) scene_replicate(primary, c);
            }
        }
    });
}

int holo_group_upload_scene(holo_group* g, const holo_scene_arrays* host) {
    return guarded_call([&] {
        check_group(g);
        require(host != nullptr, HOLO_ERR_USAGE, "null argument");
        for (auto& l : g->locals) {
            holo_ctx* primary = l.lanes[0].ctx;
            if (holo_scene_upload(primary, host) != HOLO_OK) throw Error(HOLO_ERR_CONFIG, holo_last_error());
            HC_CUDA(cudaSetDevice(l.device));
            if (g->plane_split > 1) {
                const holo_mesh m = layout(g->world, l.rank, g->plane_split, host->num_planes, 0, 0);
                scene_restrict_planes(primary, m.plane_begin, m.plane_end);
            }
            for (size_t k = 1; k < l.lanes.size(); ++k) scene_replicate(primary, l.lanes[k].ctx);
        }
    });
}

int holo_group_render(holo_group* g, const holo_camera* cams, int num_views, const holo_wave* wave,
                      const holo_raster_settings* settings, const holo_prop_options* prop, unsigned outputs,
                      unsigned flags, const holo_view_outputs* outs, holo_frame_info* infos) {
    return guarded_call([&] {
        check_group(g);
        require(cams && wave && settings, HOLO_ERR_USAGE, "null argument");
        require(num_views >= 1, HOLO_ERR_USAGE, "group: at least one view");
        const holo_prop_options po = prop ? *prop : holo_prop_options{0, 0};
        const int C = wave->channels, W = wave->nx, H = wave->ny;
        const size_t P = static_cast<size_t>(W) * H;
        const bool sharded = g->plane_split > 1 || (flags & HOLO_GROUP_SHARDED_PATH);
        const bool gather = sharded && (flags & HOLO_GROUP_GATHER_HOLOGRAM) && (outputs & HOLO_OUT_HOLOGRAM);
        require(!(sharded && po.pad2x), HOLO_ERR_CONFIG, "plane-sharded rendering does not support pad2x");
        const int nloc = static_cast<int>(g->locals.size());
        std::vector<holo_mesh> mesh(nloc);
        int steps = 0;
        for (int i = 0; i < nloc; ++i) {
            mesh[i] = layout(g->world, g->locals[i].rank, g->plane_split, wave->num_planes, num_views, C);
            steps = std::max(steps, mesh[i].view_end - mesh[i].view_begin);
        }
        if (infos)
            for (int k = 0; k < num_views * nloc; ++k) infos[k] = holo_frame_info{};
        for (int step = 0; step < steps; ++step) {
            std::vector<holo_group::Lane*> lanes;
            std::vector<int> who, views;
            for (int i = 0; i < nloc; ++i) {
                const int v = mesh[i].view_begin + step;
                if (v >= mesh[i].view_end) continue;
                auto& l = g->locals[i];
                lanes.push_back(&l.lanes[(l.frames++) % l.lanes.size()]);
                who.push_back(i);
                views.push_back(v);
            }
            auto dest = [&](size_t j) {
                holo_ctx* c = lanes[j]->ctx;
                const holo_view_outputs* o = outs ? &outs[static_cast<size_t>(views[j]) * nloc + who[j]] : nullptr;
                c->out_dest[0] = o ? o->hologram : nullptr;
                c->out_dest[1] = o ? o->replayed : nullptr;
                c->out_dest[2] = o ? o->intensities : nullptr;
            };
            auto info_of = [&](size_t j) -> holo_frame_info* {
                return infos ? &infos[static_cast<size_t>(views[j]) * nloc + who[j]] : nullptr;
            };
            try {
                if (!sharded) {
                    for (size_t j = 0; j < lanes.size(); ++j) {
                        HC_CUDA(cudaSetDevice(lanes[j]->ctx->device));
                        dest(j);
                        render_whole(lanes[j]->ctx, cams[views[j]], *wave, *settings, po, outputs, info_of(j));
                    }
                } else {
                    std::vector<cx<float>*> spec(lanes.size());
                    for (size_t j = 0; j < lanes.size(); ++j) {
                        holo_ctx* c = lanes[j]->ctx;
                        HC_CUDA(cudaSetDevice(c->device));
                        dest(j);
                        spec[j] = static_cast<cx<float>*>(c->buffer("group_spectrum", sizeof(cx<float>) * C * P));
                        const holo_mesh& m = mesh[who[j]];
                        shard_front(c, cams[views[j]], *wave, *settings, po, m.plane_begin, m.plane_end, outputs,
                                    spec[j], info_of(j));
                    }
                    for (int ch = 0; ch < C; ++ch) {
                        std::vector<float*> bufs;
                        std::vector<cudaEvent_t> ready, done;
                        for (size_t j = 0; j < lanes.size(); ++j) {
                            bufs.push_back(reinterpret_cast<float*>(spec[j] + static_cast<size_t>(ch) * P));
                            ready.push_back(lanes[j]->ctx->ev_chan_ready[ch]);
                            done.push_back(lanes[j]->ctx->ev_chan_done[ch]);
                        }
                        plane_sum(g, lanes, who, bufs, 2 * P, ready, done);
                    }
                    for (size_t j = 0; j < lanes.size(); ++j) {
                        holo_ctx* c = lanes[j]->ctx;
                        HC_CUDA(cudaSetDevice(c->device));
                        const holo_mesh& m = mesh[who[j]];
                        shard_back(c, *wave, po, m.plane_begin, m.plane_end, spec[j], outputs, m.holo_channels);
                    }
                    if (gather) {
                        // every rank of the plane group receives all channels: the
                        // channels formed elsewhere are zeroed here, then summed
                        std::vector<float*> bufs;
                        std::vector<cudaEvent_t> ready, done;
                        for (size_t j = 0; j < lanes.size(); ++j) {
                            holo_ctx* c = lanes[j]->ctx;
                            HC_CUDA(cudaSetDevice(c->device));
                            cx<float>* h = frame_hologram(c, C, P);
                            for (int ch = 0; ch < C; ++ch)
                                if (!((mesh[who[j]].holo_channels >> ch) & 1u))
                                    HC_CUDA(cudaMemsetAsync(h + static_cast<size_t>(ch) * P, 0, sizeof(cx<float>) * P,
                                                            c->stream));
                            c->f_outputs |= HOLO_OUT_HOLOGRAM;
                            HC_CUDA(cudaEventRecord(lanes[j]->ev_holo, c->stream));
                            bufs.push_back(reinterpret_cast<float*>(h));
                            ready.push_back(lanes[j]->ev_holo);
                            done.push_back(c->ev_chan_done[0]);
                        }
                        plane_sum(g, lanes, who, bufs, 2 * static_cast<size_t>(C) * P, ready, done);
                        for (size_t j = 0; j < lanes.size(); ++j)
                            HC_CUDA(cudaStreamWaitEvent(lanes[j]->ctx->stream, lanes[j]->ctx->ev_chan_done[0], 0));
                    }
                }
            } catch (...) {
                for (auto* ln : lanes) std::fill(std::begin(ln->ctx->out_dest), std::end(ln->ctx->out_dest), nullptr);
                throw;
            }
            for (auto* ln : lanes) std::fill(std::begin(ln->ctx->out_dest), std::end(ln->ctx->out_dest), nullptr);
        }
    });
}

int holo_group_set_async(holo_group* g, int enable) {
    return guarded_call([&] {
        check_group(g);
        for (auto& l : g->locals) {
            size_t cap = 0;
            for (auto& ln : l.lanes) cap = std::max(cap, ln.ctx->e_cap);
            for (auto& ln : l.lanes) {
                if (enable && holo_ctx_reserve_entries(ln.ctx, cap) != HOLO_OK)
                    throw Error(HOLO_ERR_USAGE, holo_last_error());
                if (holo_ctx_set_async(ln.ctx, enable) != HOLO_OK) throw Error(HOLO_ERR_USAGE, holo_last_error());
            }
        }
    });
}

int holo_group_frame_status(holo_group* g) {
    int rc = HOLO_OK;
    std::string msg;
    if (!g) return guarded_call([] { throw Error(HOLO_ERR_USAGE, "null group"); });
    for (auto& l : g->locals)
        for (auto& ln : l.lanes) {
            const int r = holo_ctx_frame_status(ln.ctx, nullptr);
            if (r != HOLO_OK && rc == HOLO_OK) {
                rc = r;
                msg = holo_last_error();
            }
        }
    if (rc != HOLO_OK) set_last_error(msg.c_str());
    return rc;
}

int holo_group_join(holo_group* g, int local, void* stream) {
    return guarded_call([&] {
        check_group(g);
        require(local >= 0 && local < static_cast<int>(g->locals.size()), HOLO_ERR_USAGE, "group: no such local rank");
        auto& l = g->locals[local];
        HC_CUDA(cudaSetDevice(l.device));
        const cudaStream_t to = static_cast<cudaStream_t>(stream);
        for (auto& ln : l.lanes) {
            for (cudaStream_t from : {ln.ctx->stream, ln.comm}) {
                if (from == to) continue;
                HC_CUDA(cudaEventRecord(ln.ev_holo, from));
                HC_CUDA(cudaStreamWaitEvent(to, ln.ev_holo, 0));
            }
        }
    });
}

uint64_t holo_group_launch_count(const holo_group* g) {
    uint64_t n = 0;
    if (g)
        for (auto& l : g->locals)
            for (auto& ln : l.lanes) n += ln.ctx->launches;
    return n;
}

int holo_group_synchronize(holo_group* g) {
    return guarded_call([&] {
        check_group(g);
        for (auto& l : g->locals) {
            HC_CUDA(cudaSetDevice(l.device));
            for (auto& ln : l.lanes) {
                HC_CUDA(cudaStreamSynchronize(ln.comm));
                HC_CUDA(cudaStreamSynchronize(ln.ctx->stream));
            }
        }
    });
}

}  // extern "C"
