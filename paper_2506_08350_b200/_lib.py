"""ctypes binding of libholo_cuda.so (include/holo_cuda.h).

The product path: every call goes to the in-tree sm_100a library.  There is no
CPU fallback -- if the library is missing or no CUDA device is visible the
call raises ``HoloError`` loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HOLO_CUDA_LIB: another build of the same library (measurement variants)
LIB_PATH = os.environ.get("HOLO_CUDA_LIB") or os.path.join(HERE, "lib", "libholo_cuda.so")
MAX_CH = 16

OK, ERR_CONFIG, ERR_IO, ERR_USAGE, ERR_NUMERIC, ERR_CUDA, ERR_OOM, ERR_NCCL = range(8)
KIND = {ERR_CONFIG: "config", ERR_IO: "io", ERR_USAGE: "usage", ERR_NUMERIC: "numeric", ERR_CUDA: "cuda",
        ERR_OOM: "oom", ERR_NCCL: "nccl"}
F32, F64 = 0, 1

OUT_LAYERS, OUT_HOLOGRAM, OUT_REPLAYED, OUT_INTENSITY, OUT_AUX, OUT_LISTS, OUT_PROJECTED = (1 << i for i in range(7))
(BUF_LAYERS, BUF_HOLOGRAM, BUF_REPLAYED, BUF_INTENSITY, BUF_T_FINAL, BUF_N_CONTRIB, BUF_ENTRY_GIDX,
 BUF_ENTRY_DEPTH, BUF_BUCKET_START, BUF_PROJECTED, BUF_RHO, BUF_TOUCHED, BUF_SPECTRUM) = range(13)

# stage ids of holo_ctx_stage_times (include/holo_cuda.h); the fft passes are, on the
# compile-time-plan path: column FFT, row pass (spectrum + inverse rows), row replay
# (sharded only), column IFFT + epilogue
STAGES = ("preprocess", "binning", "composite", "fft_pass1", "fft_pass2", "fft_pass3", "fft_pass4")


class HoloError(RuntimeError):
    """Mirror of holo::HoloError (proj/include/holo/common.hpp:76-79)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


class Wave(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("pitch", C.c_double), ("channels", C.c_int),
                ("wavelengths", C.c_double * MAX_CH), ("distance", C.c_double), ("volume_depth", C.c_double),
                ("num_planes", C.c_int)]


class Camera(C.Structure):
    _fields_ = [("pose", C.c_double * 6), ("focal_px", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int), ("height", C.c_int)]


class RasterSettings(C.Structure):
    _fields_ = [("near_clip", C.c_double), ("dilation", C.c_double), ("plane_eps", C.c_double),
                ("term_eps", C.c_double), ("alpha_floor", C.c_double), ("alpha_clamp", C.c_double),
                ("radius_form_cap", C.c_double), ("ste_tau", C.c_double), ("soft_assignment", C.c_int),
                ("soft_tau", C.c_double), ("tile", C.c_int)]


class PropOptions(C.Structure):
    _fields_ = [("pad2x", C.c_int), ("local_band_limit", C.c_int)]


_dp = C.POINTER(C.c_double)


class SceneArrays(C.Structure):
    _fields_ = [("n", C.c_size_t), ("num_planes", C.c_int), ("positions", C.c_void_p), ("rotations", C.c_void_p),
                ("log_scales", C.c_void_p), ("amplitudes", C.c_void_p), ("opacity_logits", C.c_void_p),
                ("phases", C.c_void_p), ("plane_logits", C.c_void_p)]


class Projected(C.Structure):
    _fields_ = [("valid", C.c_int32), ("n", C.c_int32), ("mu_x", C.c_double), ("mu_y", C.c_double),
                ("inv00", C.c_double), ("inv01", C.c_double), ("inv11", C.c_double), ("radius", C.c_double),
                ("xc", C.c_double), ("yc", C.c_double), ("zc", C.c_double), ("alpha_sig", C.c_double),
                ("amp", C.c_double * 3), ("phase", C.c_double * 3), ("plane", C.c_int32), ("pad_", C.c_int32)]


GRAD_FIELDS = ("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases", "plane_logits",
               "mu_screen")


class SceneGrads(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in GRAD_FIELDS]


class LossOptions(C.Structure):
    _fields_ = [("lambda_ssim", C.c_double), ("lambda_opacity", C.c_double), ("use_plain_mse", C.c_int)]


class LossBreakdown(C.Structure):
    _fields_ = [("total", C.c_double), ("recon", C.c_double), ("ssim", C.c_double), ("opacity", C.c_double),
                ("psnr_mean", C.c_double)]


OPTIM_FIELDS = ("lr_positions", "lr_rotations", "lr_log_scales", "lr_amplitudes", "lr_phases", "lr_opacities",
                "lr_plane_logits", "beta1", "beta2", "beta3", "eps")


class OptimizerConfig(C.Structure):
    _fields_ = [(k, C.c_double) for k in OPTIM_FIELDS] + [("use_adam", C.c_int), ("schedule_total", C.c_longlong),
                                                          ("lr_floor", C.c_double)]


class PhaseOptions(C.Structure):
    _fields_ = [("lambda_ssim", C.c_double), ("prop", PropOptions), ("use_adam", C.c_int)]


class FrameInfo(C.Structure):
    _fields_ = [("num_entries", C.c_uint64), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
                ("num_buckets", C.c_int32), ("max_bucket", C.c_int32), ("num_valid", C.c_int32),
                ("pad_", C.c_int32)]


class Mesh(C.Structure):
    """holo_mesh: a rank's coordinates in the (view groups x plane split) mesh."""
    _fields_ = [("world", C.c_int), ("rank", C.c_int), ("plane_split", C.c_int), ("view_groups", C.c_int),
                ("plane_rank", C.c_int), ("view_group", C.c_int), ("plane_begin", C.c_int), ("plane_end", C.c_int),
                ("view_begin", C.c_int), ("view_end", C.c_int), ("holo_channels", C.c_uint)]


class ViewOutputs(C.Structure):
    _fields_ = [("hologram", C.c_void_p), ("replayed", C.c_void_p), ("intensities", C.c_void_p)]


GROUP_ID_BYTES = 128
GROUP_GATHER_HOLOGRAM, GROUP_SHARDED_PATH = 1, 2
# int fn(void* user, float* device_buffer, size_t count, void* cuda_stream)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)

_LIB = None


def lib() -> C.CDLL:
    """Load libholo_cuda.so once; raise loudly if it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise HoloError("usage", f"libholo_cuda.so not built at {LIB_PATH}; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    vp, i, u, d, sz = C.c_void_p, C.c_int, C.c_uint, C.c_double, C.c_size_t
    P = C.POINTER
    sig = {
        "holo_last_error": (C.c_char_p, []),
        "holo_abi_version": (i, []),
        "holo_fft_supported": (i, [i]),
        "holo_ctx_create": (i, [i, P(vp)]),
        "holo_ctx_destroy": (i, [vp]),
        "holo_ctx_set_stream": (i, [vp, vp]),
        "holo_ctx_use_own_stream": (i, [vp]),
        "holo_ctx_get_stream": (vp, [vp]),
        "holo_ctx_get_copy_stream": (vp, [vp, i]),
        "holo_ctx_synchronize": (i, [vp]),
        "holo_ctx_enable_timing": (i, [vp, i]),
        "holo_ctx_stage_times": (i, [vp, P(d), P(i), i]),
        "holo_ctx_reset_timing": (i, [vp]),
        "holo_ctx_launch_count": (C.c_uint64, [vp]),
        "holo_ctx_set_guard": (i, [vp, i]),
        "holo_ctx_check_guards": (i, [vp]),
        "holo_ctx_set_async": (i, [vp, i]),
        "holo_ctx_reserve_entries": (i, [vp, C.c_uint64]),
        "holo_ctx_frame_status": (i, [vp, P(FrameInfo)]),
        "holo_scene_upload": (i, [vp, P(SceneArrays)]),
        "holo_scene_upload_device": (i, [vp, P(SceneArrays)]),
        "holo_render": (i, [vp, P(Camera), P(Wave), P(RasterSettings), P(PropOptions), u, P(FrameInfo)]),
        "holo_render_begin": (i, [vp, P(Camera), P(Wave), P(RasterSettings), P(PropOptions), i, i, vp, u,
                                  P(FrameInfo)]),
        "holo_render_end": (i, [vp, P(Wave), P(PropOptions), i, i, vp, u]),
        "holo_brute_force_forward": (i, [vp, P(Camera), P(Wave), P(RasterSettings)]),
        "holo_frame_buffer": (i, [vp, i, P(vp), P(sz)]),
        "holo_frame_download": (i, [vp, i, vp, sz]),
        "holo_frame_download_async": (i, [vp, i, vp, sz]),
        "holo_raster_backward": (i, [vp, P(Camera), P(Wave), P(RasterSettings), vp, P(SceneGrads)]),
        "holo_pipeline_backward": (i, [vp, P(Camera), P(Wave), P(RasterSettings), P(PropOptions), vp,
                                       P(SceneGrads), vp, vp]),
        "holo_losses": (i, [vp, vp, vp, vp, i, i, i, i, P(LossOptions), P(LossBreakdown), P(d), vp]),
        "holo_total_loss": (i, [vp, P(Camera), P(Wave), P(RasterSettings), P(PropOptions), P(LossOptions), vp, vp,
                                P(LossBreakdown), P(d), P(SceneGrads)]),
        "holo_optim_create": (i, [vp, P(vp)]),
        "holo_optim_destroy": (i, [vp]),
        "holo_optim_step": (i, [vp, vp, P(SceneGrads), P(OptimizerConfig), P(i)]),
        "holo_optim_counts": (i, [vp, P(C.c_longlong), P(C.c_longlong)]),
        "holo_scene_download": (i, [vp, P(SceneArrays)]),
        "holo_phase_only_loss": (i, [vp, vp, vp, P(Wave), P(PhaseOptions), P(d), vp]),
        "holo_convert_phase_only": (i, [vp, vp, P(Wave), i, d, P(PhaseOptions), vp, vp, P(d)]),
        "holo_fft2": (i, [vp, vp, i, i, i, i, i]),
        "holo_transfer_function": (i, [vp, P(Wave), d, P(PropOptions), vp, i]),
        "holo_propagate": (i, [vp, vp, vp, i, i, i, P(Wave), d, P(PropOptions), i]),
        "holo_forward_record": (i, [vp, vp, i, vp, P(Wave), P(PropOptions), i]),
        "holo_inverse_propagate": (i, [vp, vp, vp, P(Wave), P(PropOptions), i]),
        "holo_intensity": (i, [vp, vp, vp, sz, i]),
        "holo_mesh_layout": (i, [i, i, i, i, i, i, P(Mesh)]),
        "holo_group_unique_id": (i, [C.c_char_p]),
        "holo_group_init_rank": (i, [vp, C.c_char_p, i, i, i, P(vp)]),
        "holo_group_init_callback": (i, [vp, i, i, i, ALLREDUCE_FN, vp, P(vp)]),
        "holo_group_create": (i, [P(i), i, i, P(vp)]),
        "holo_group_destroy": (i, [vp]),
        "holo_group_local_count": (i, [vp]),
        "holo_group_context": (i, [vp, i, P(vp)]),
        "holo_group_mesh": (i, [vp, i, i, i, i, P(Mesh)]),
        "holo_group_set_lanes": (i, [vp, i]),
        "holo_group_upload_scene": (i, [vp, P(SceneArrays)]),
        "holo_group_render": (i, [vp, P(Camera), i, P(Wave), P(RasterSettings), P(PropOptions), u, u,
                                  P(ViewOutputs), P(FrameInfo)]),
        "holo_group_synchronize": (i, [vp]),
        "holo_group_set_async": (i, [vp, i]),
        "holo_group_frame_status": (i, [vp]),
        "holo_group_join": (i, [vp, i, vp]),
        "holo_group_launch_count": (C.c_uint64, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _LIB = L
    return L


def check(rc: int) -> None:
    if rc != OK:
        msg = lib().holo_last_error().decode()
        raise HoloError(KIND.get(rc, "numeric"), msg)
