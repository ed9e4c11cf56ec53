"""Host-side mirror of the reference render/propagate API over libholo_cuda.

Function names, arguments and errors follow proj/include/holo/*.hpp:

* raster_forward(scene, cam, cfg, settings)      rasterizer.hpp:75-76
* pipeline_forward(scene, cam, cfg, opt)         pipeline.hpp:41-42
* propagate(u, cfg, z, opt)                      propagation.hpp:31
* forward_record(layers, cfg, opt)               propagation.hpp:35-36
* inverse_propagate(hologram, cfg, opt)          propagation.hpp:39-40
* transfer_function(cfg, z, opt)                 propagation.hpp:27
* fft2 / ifft2                                   fft.hpp:11-12
* intensity(u)                                   field.hpp:45
* raster_backward / pipeline_backward            rasterizer.hpp:79-81, pipeline.cpp:63-91
* losses(I, I_gt, masks, opt)                    losses.hpp (loss_recon / loss_mse, loss_ssim, psnr)
* total_loss(scene, cam, cfg, target, opt)       pipeline.hpp:54-56
* Optimizer(ctx).step(grads, cfg)                optimizer.hpp:55-58 (optimizer_step)
* phase_only_loss / convert_phase_only /
  phase_gradient_oracle                          phase_only.hpp:39-62

Host data is numpy (complex128 fields [C, H, W], like the reference's f64
ComplexField); every call runs on the GPU through the C-ABI.  The render path
computes in fp32 (complex64) as the north star specifies; the propagation
operators take ``precision="f64"`` (default, reference precision) or "f32".

``Context`` is the device-resident interface used by bench.py and the sharded
renderer: scene stays in HBM, outputs stay in context buffers and are exposed
as zero-copy torch views.
"""
from __future__ import annotations

import ctypes as C
from typing import Iterable, List, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import HoloError
from .holotypes import (CameraView, GaussianScene, LossBreakdown, OptimizerConfig, PhaseOnlyHologram, PhaseOnlyOptions,
                        PhaseOnlyResult, PipelineForward, PipelineOptions, PropagationOptions, RasterForward,
                        RenderSettings, WaveConfig, plane_positions)

_NP = {"f32": (L.F32, np.complex64, np.float32), "f64": (L.F64, np.complex128, np.float64)}


def _wave(cfg: WaveConfig) -> L.Wave:
    w = L.Wave()
    w.nx, w.ny = int(cfg.nx), int(cfg.ny)
    w.pitch = float(cfg.pitch)
    wl = list(cfg.wavelengths)
    if len(wl) > L.MAX_CH:
        raise HoloError("config", "too many wavelength channels")
    w.channels = len(wl)
    for i, v in enumerate(wl):
        w.wavelengths[i] = float(v)
    w.distance = float(cfg.distance)
    w.volume_depth = float(cfg.volume_depth)
    w.num_planes = int(cfg.num_planes)
    return w


def _camera(cam: CameraView) -> L.Camera:
    c = L.Camera()
    for i in range(6):
        c.pose[i] = float(cam.pose[i])
    c.focal_px = float(cam.focal_px)
    c.cx, c.cy = float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def _settings(st: Optional[RenderSettings]) -> L.RasterSettings:
    st = st or RenderSettings()
    s = L.RasterSettings()
    for k in ("near_clip", "dilation", "plane_eps", "term_eps", "alpha_floor", "alpha_clamp", "radius_form_cap",
              "ste_tau", "soft_tau"):
        setattr(s, k, float(getattr(st, k)))
    s.soft_assignment = int(bool(st.soft_assignment))
    s.tile = int(st.tile)
    return s


def _loss_opts(opt: Optional[PipelineOptions]) -> L.LossOptions:
    opt = opt or PipelineOptions()
    o = L.LossOptions()
    o.lambda_ssim = float(opt.lambda_ssim)
    o.lambda_opacity = float(opt.lambda_opacity)
    o.use_plain_mse = int(bool(opt.use_plain_mse))
    return o


def _optim_cfg(cfg: Optional[OptimizerConfig]) -> L.OptimizerConfig:
    cfg = cfg or OptimizerConfig()
    c = L.OptimizerConfig()
    for k in L.OPTIM_FIELDS + ("lr_floor",):
        setattr(c, k, float(getattr(cfg, k)))
    c.use_adam = int(bool(cfg.use_adam))
    c.schedule_total = int(cfg.schedule_total)
    return c


def _breakdown(b: L.LossBreakdown, psnr) -> LossBreakdown:
    return LossBreakdown(total=b.total, recon=b.recon, ssim=b.ssim, opacity=b.opacity, psnr_mean=b.psnr_mean,
                         psnr=[float(x) for x in psnr])


def _phase_opts(opt: Optional[PhaseOnlyOptions]) -> L.PhaseOptions:
    opt = opt or PhaseOnlyOptions()
    o = L.PhaseOptions()
    o.lambda_ssim = float(opt.lambda_ssim)
    o.prop = _prop(opt.prop)
    o.use_adam = int(bool(opt.use_adam))
    return o


def _prop(opt: Optional[PropagationOptions]) -> L.PropOptions:
    opt = opt or PropagationOptions()
    p = L.PropOptions()
    p.pad2x = int(bool(opt.pad2x))
    p.local_band_limit = int(bool(opt.local_band_limit))
    return p


class _CudaArray:
    """Zero-copy __cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _torch():
    import torch  # plumbing only: device memory, streams, collectives

    if not torch.cuda.is_available():
        raise HoloError("usage", "no CUDA device visible; libholo_cuda has no CPU fallback")
    return torch


class Context:
    """One holo_ctx: a CUDA stream (torch's current stream by default), the resident
    scene and the last frame's outputs."""

    def __init__(self, device: int = 0, use_torch_stream: bool = True):
        torch = _torch()
        self.device = device
        self.lib = L.lib()
        h = C.c_void_p()
        L.check(self.lib.holo_ctx_create(device, C.byref(h)))
        self.h = h
        self.info = L.FrameInfo()
        self._keep = []
        if use_torch_stream:
            with torch.cuda.device(device):
                self.set_stream(torch.cuda.current_stream().cuda_stream)

    def close(self):
        if getattr(self, "h", None):
            L.check(self.lib.holo_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------- plumbing
    def set_stream(self, stream: int) -> None:
        """Enqueue on this CUDA stream handle (0 = the legacy default stream)."""
        L.check(self.lib.holo_ctx_set_stream(self.h, C.c_void_p(stream or None)))

    def use_own_stream(self) -> None:
        L.check(self.lib.holo_ctx_use_own_stream(self.h))

    def stream(self) -> int:
        return int(self.lib.holo_ctx_get_stream(self.h) or 0)

    def copy_stream(self, which: int) -> int:
        """Copy stream handle: 0 = host uploads, 1 = asynchronous downloads."""
        return int(self.lib.holo_ctx_get_copy_stream(self.h, int(which)) or 0)

    def synchronize(self) -> None:
        L.check(self.lib.holo_ctx_synchronize(self.h))

    def launch_count(self) -> int:
        return int(self.lib.holo_ctx_launch_count(self.h))

    def set_guard(self, on: bool = True) -> None:
        """Guard bands after every scratch buffer (set before the first render)."""
        L.check(self.lib.holo_ctx_set_guard(self.h, int(on)))

    def check_guards(self) -> None:
        """Raise HoloError naming any scratch buffer whose guard band was overwritten."""
        L.check(self.lib.holo_ctx_check_guards(self.h))

    def set_async(self, on: bool = True) -> None:
        """Asynchronous frames: render() only enqueues; frame_status() reports (holo_cuda.h)."""
        L.check(self.lib.holo_ctx_set_async(self.h, int(on)))

    def reserve_entries(self, n: int) -> None:
        L.check(self.lib.holo_ctx_reserve_entries(self.h, int(n)))

    def frame_status(self) -> L.FrameInfo:
        """Wait for this context's frames; raise on flags raised since the last call."""
        L.check(self.lib.holo_ctx_frame_status(self.h, C.byref(self.info)))
        return self.info

    def enable_timing(self, on: bool = True) -> None:
        L.check(self.lib.holo_ctx_enable_timing(self.h, int(on)))

    def reset_timing(self) -> None:
        L.check(self.lib.holo_ctx_reset_timing(self.h))

    def stage_times(self) -> dict:
        ms = (C.c_double * 8)()
        n = (C.c_int * 8)()
        L.check(self.lib.holo_ctx_stage_times(self.h, ms, n, 8))
        return {name: (ms[i], n[i]) for i, name in enumerate(L.STAGES)}

    # ---------------------------------------------------------------- scene
    def upload_scene(self, scene: GaussianScene) -> None:
        """Host f64 arrays -> HBM (validated on the device at render time, scene.cpp:19-32)."""
        n = scene.size()
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (scene.positions, scene.rotations, scene.log_scales, scene.amplitudes, scene.opacity_logits,
                 scene.phases, scene.plane_logits)]
        sizes = [a.size for a in arrs]
        if sizes != [3 * n, 4 * n, 3 * n, 3 * n, n, 3 * n, n * scene.num_planes]:
            raise HoloError("config", "scene arrays have inconsistent sizes")
        s = L.SceneArrays()
        s.n, s.num_planes = n, int(scene.num_planes)
        for name, a in zip(("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases",
                            "plane_logits"), arrs):
            setattr(s, name, a.ctypes.data)
        L.check(self.lib.holo_scene_upload(self.h, C.byref(s)))
        # pageable host memory: the copy has completed when the call returns; keep
        # the arrays alive until the stream drains anyway
        self._keep = arrs

    def upload_scene_pointers(self, n: int, num_planes: int, ptrs: Sequence[int], device: bool) -> None:
        """Scene arrays given as raw pointers (pinned host or device), in reference order."""
        s = L.SceneArrays()
        s.n, s.num_planes = int(n), int(num_planes)
        for name, p in zip(("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases",
                            "plane_logits"), ptrs):
            setattr(s, name, int(p))
        fn = self.lib.holo_scene_upload_device if device else self.lib.holo_scene_upload
        L.check(fn(self.h, C.byref(s)))

    # --------------------------------------------------------------- render
    def render(self, cam: CameraView, cfg: WaveConfig, settings: Optional[RenderSettings] = None,
               prop: Optional[PropagationOptions] = None,
               outputs: int = L.OUT_HOLOGRAM | L.OUT_INTENSITY) -> L.FrameInfo:
        L.check(self.lib.holo_render(self.h, C.byref(_camera(cam)), C.byref(_wave(cfg)),
                                     C.byref(_settings(settings)), C.byref(_prop(prop)), int(outputs),
                                     C.byref(self.info)))
        return self.info

    def render_begin(self, cam, cfg, settings, prop, plane_begin, plane_end, spectrum_ptr: int, outputs: int):
        L.check(self.lib.holo_render_begin(self.h, C.byref(_camera(cam)), C.byref(_wave(cfg)),
                                           C.byref(_settings(settings)), C.byref(_prop(prop)), int(plane_begin),
                                           int(plane_end), C.c_void_p(spectrum_ptr or None), int(outputs),
                                           C.byref(self.info)))
        return self.info

    def render_end(self, cfg, prop, plane_begin, plane_end, spectrum_ptr: int, outputs: int):
        L.check(self.lib.holo_render_end(self.h, C.byref(_wave(cfg)), C.byref(_prop(prop)), int(plane_begin),
                                         int(plane_end), C.c_void_p(spectrum_ptr or None), int(outputs)))

    # ------------------------------------------------------------- gradients
    def _grad_tensors(self, n: int, num_planes: int):
        torch = _torch()
        shapes = {"positions": (n, 3), "rotations": (n, 4), "log_scales": (n, 3), "amplitudes": (n, 3),
                  "opacity_logits": (n,), "phases": (n, 3), "plane_logits": (n, num_planes), "mu_screen": (n, 2)}
        out = {k: torch.empty(shapes[k], dtype=torch.float64, device=f"cuda:{self.device}") for k in L.GRAD_FIELDS}
        g = L.SceneGrads()
        for k in L.GRAD_FIELDS:
            setattr(g, k, out[k].data_ptr())
        return g, out

    def raster_backward(self, cam: CameraView, cfg: WaveConfig, settings: Optional[RenderSettings],
                        grad_layers, n: int):
        """raster_backward (rasterizer.cpp:332-528) of this context's last render
        (outputs must include OUT_AUX).  grad_layers: device complex64 tensor
        [L, C, H, W].  Returns a dict of f64 device tensors (SceneGradients)."""
        g, out = self._grad_tensors(n, cfg.num_planes)
        L.check(self.lib.holo_raster_backward(self.h, C.byref(_camera(cam)), C.byref(_wave(cfg)),
                                              C.byref(_settings(settings)), C.c_void_p(grad_layers.data_ptr()),
                                              C.byref(g)))
        return out

    def pipeline_backward(self, cam: CameraView, cfg: WaveConfig, settings: Optional[RenderSettings],
                          prop: Optional[PropagationOptions], grad_intensities, n: int):
        """The gradient branch of total_loss (pipeline.cpp:63-80) for dL/dI (device
        float32 tensor [L, C, H, W]) of the last render (outputs must include
        OUT_REPLAYED | OUT_AUX).  Returns (grads, grad_layers, grad_hologram)."""
        torch = _torch()
        Cn, H, W = cfg.channels(), cfg.ny, cfg.nx
        gl = torch.empty((cfg.num_planes, Cn, H, W), dtype=torch.complex64, device=f"cuda:{self.device}")
        gh = torch.empty((Cn, H, W), dtype=torch.complex64, device=f"cuda:{self.device}")
        g, out = self._grad_tensors(n, cfg.num_planes)
        L.check(self.lib.holo_pipeline_backward(self.h, C.byref(_camera(cam)), C.byref(_wave(cfg)),
                                                C.byref(_settings(settings)), C.byref(_prop(prop)),
                                                C.c_void_p(grad_intensities.data_ptr()), C.byref(g),
                                                C.c_void_p(gl.data_ptr()), C.c_void_p(gh.data_ptr())))
        return out, gl, gh

    # ---------------------------------------------------------- training step
    def losses(self, intensities, targets, masks, opt: Optional[PipelineOptions] = None, grad: bool = True):
        """loss_recon (or loss_mse) + loss_ssim + psnr (losses.cpp) over device f64
        tensors [L, C, H, W] (masks [L, H, W]).  Returns (LossBreakdown, dL/dI or None)."""
        torch = _torch()
        Ln, Cn, H, W = (int(x) for x in intensities.shape)
        b = L.LossBreakdown()
        psnr = (C.c_double * Ln)()
        g = torch.empty_like(intensities) if grad else None
        L.check(self.lib.holo_losses(self.h, C.c_void_p(intensities.data_ptr()), C.c_void_p(targets.data_ptr()),
                                     C.c_void_p(masks.data_ptr() if masks is not None else None), Ln, Cn, H, W,
                                     C.byref(_loss_opts(opt)), C.byref(b), psnr,
                                     C.c_void_p(g.data_ptr() if g is not None else None)))
        return _breakdown(b, psnr), g

    def total_loss(self, cam: CameraView, cfg: WaveConfig, targets, masks, opt: Optional[PipelineOptions] = None,
                   n: Optional[int] = None):
        """total_loss (pipeline.cpp:30-95) on the resident scene; targets / masks are
        device f64 tensors [L, C, H, W] / [L, H, W].  With n (the scene size) the
        gradients are computed and returned as a dict of f64 device tensors."""
        opt = opt or PipelineOptions()
        b = L.LossBreakdown()
        psnr = (C.c_double * cfg.num_planes)()
        g = out = None
        if n is not None:
            g, out = self._grad_tensors(n, cfg.num_planes)
        L.check(self.lib.holo_total_loss(self.h, C.byref(_camera(cam)), C.byref(_wave(cfg)),
                                         C.byref(_settings(opt.raster)), C.byref(_prop(opt.prop)),
                                         C.byref(_loss_opts(opt)), C.c_void_p(targets.data_ptr()),
                                         C.c_void_p(masks.data_ptr() if masks is not None else None), C.byref(b),
                                         psnr, C.byref(g) if g is not None else None))
        return _breakdown(b, psnr), out

    # ------------------------------------------------------- phase-only conversion
    def phase_only_loss(self, P, theta, cfg: WaveConfig, opt: Optional[PhaseOnlyOptions] = None, grad=None) -> float:
        """phase_only_loss on device tensors: P complex128 [C, H, W], theta f64 [C, H, W];
        grad (f64 tensor, optional) receives d loss / d theta."""
        loss = C.c_double()
        L.check(self.lib.holo_phase_only_loss(self.h, C.c_void_p(P.data_ptr()), C.c_void_p(theta.data_ptr()),
                                              C.byref(_wave(cfg)), C.byref(_phase_opts(opt)), C.byref(loss),
                                              C.c_void_p(grad.data_ptr() if grad is not None else None)))
        return loss.value

    def convert_phase_only(self, P, cfg: WaveConfig, iters: int = 1000, lr: float = 0.02,
                           opt: Optional[PhaseOnlyOptions] = None, theta0=None):
        """convert_phase_only on a device complex128 tensor: (best phase tensor, trace)."""
        torch = _torch()
        out = torch.empty(P.shape, dtype=torch.float64, device=P.device)
        trace = (C.c_double * (max(int(iters), 0) + 1))()
        L.check(self.lib.holo_convert_phase_only(self.h, C.c_void_p(P.data_ptr()), C.byref(_wave(cfg)), int(iters),
                                                 float(lr), C.byref(_phase_opts(opt)),
                                                 C.c_void_p(theta0.data_ptr() if theta0 is not None else None),
                                                 C.c_void_p(out.data_ptr()), trace))
        return out, list(trace)

    def download_scene(self, n: int, num_planes: int) -> GaussianScene:
        """The resident scene back on the host (checkpointing after optimizer steps)."""
        arrs = {"positions": np.empty((n, 3)), "rotations": np.empty((n, 4)), "log_scales": np.empty((n, 3)),
                "amplitudes": np.empty((n, 3)), "opacity_logits": np.empty((n,)), "phases": np.empty((n, 3)),
                "plane_logits": np.empty((n, num_planes))}
        s = L.SceneArrays()
        s.n, s.num_planes = int(n), int(num_planes)
        for k, a in arrs.items():
            setattr(s, k, a.ctypes.data)
        L.check(self.lib.holo_scene_download(self.h, C.byref(s)))
        return GaussianScene(num_planes=int(num_planes), **arrs)

    def buffer(self, which: int):
        p = C.c_void_p()
        n = C.c_size_t()
        L.check(self.lib.holo_frame_buffer(self.h, int(which), C.byref(p), C.byref(n)))
        return int(p.value or 0), int(n.value)

    def download(self, which: int, dtype, shape) -> np.ndarray:
        out = np.empty(shape, dtype=dtype)
        L.check(self.lib.holo_frame_download(self.h, int(which), out.ctypes.data, out.nbytes))
        return out

    def download_into(self, which: int, host_ptr: int, nbytes: int, wait: bool = True) -> None:
        """Copy an output buffer to host memory; wait=False only enqueues it on the
        context stream (pinned memory; complete after synchronize())."""
        fn = self.lib.holo_frame_download if wait else self.lib.holo_frame_download_async
        L.check(fn(self.h, int(which), C.c_void_p(host_ptr), int(nbytes)))

    def tensor(self, which: int, dtype: str, shape):
        """Zero-copy torch view of an output buffer (valid until the next render)."""
        torch = _torch()
        ptr, nbytes = self.buffer(which)
        typestr = {"c8": "<c8", "f4": "<f4", "i4": "<i4", "u4": "<u4", "f8": "<f8", "u1": "|u1"}[dtype]
        return torch.as_tensor(_CudaArray(ptr, shape, typestr), device=f"cuda:{self.device}")

    # ------------------------------------------------------------ operators
    def _dev(self, arr: np.ndarray, precision: str):
        torch = _torch()
        _, cdt, _ = _NP[precision]
        a = np.ascontiguousarray(arr, dtype=cdt)
        return torch.from_numpy(a).to(f"cuda:{self.device}")

    def fft2(self, data: np.ndarray, inverse: bool = False, precision: str = "f64") -> np.ndarray:
        d = self._dev(data, precision)
        h, w = d.shape[-2:]
        batch = int(np.prod(d.shape[:-2])) if d.dim() > 2 else 1
        L.check(self.lib.holo_fft2(self.h, d.data_ptr(), w, h, batch, int(inverse), _NP[precision][0]))
        return d.cpu().numpy()

    def transfer_function(self, cfg: WaveConfig, z: float, opt=None, precision: str = "f64") -> np.ndarray:
        torch = _torch()
        f = 2 if (opt and opt.pad2x) else 1
        out = torch.empty((cfg.channels(), cfg.ny * f, cfg.nx * f),
                          dtype=torch.complex64 if precision == "f32" else torch.complex128,
                          device=f"cuda:{self.device}")
        L.check(self.lib.holo_transfer_function(self.h, C.byref(_wave(cfg)), float(z), C.byref(_prop(opt)),
                                                out.data_ptr(), _NP[precision][0]))
        return out.cpu().numpy()

    def propagate(self, u: np.ndarray, cfg: WaveConfig, z: float, opt=None, precision: str = "f64") -> np.ndarray:
        d = self._dev(u, precision)
        if d.dim() != 3:
            raise HoloError("config", "propagate: field does not match the configured grid")
        c, h, w = d.shape
        out = d.new_empty(d.shape)
        L.check(self.lib.holo_propagate(self.h, d.data_ptr(), out.data_ptr(), w, h, c, C.byref(_wave(cfg)),
                                        float(z), C.byref(_prop(opt)), _NP[precision][0]))
        return out.cpu().numpy()

    def forward_record(self, layers, cfg: WaveConfig, opt=None, precision: str = "f64") -> np.ndarray:
        d = self._dev(np.stack([np.asarray(x) for x in layers]), precision)
        out = d.new_empty(d.shape[1:])
        L.check(self.lib.holo_forward_record(self.h, d.data_ptr(), d.shape[0], out.data_ptr(), C.byref(_wave(cfg)),
                                             C.byref(_prop(opt)), _NP[precision][0]))
        return out.cpu().numpy()

    def inverse_propagate(self, hologram: np.ndarray, cfg: WaveConfig, opt=None, precision: str = "f64"):
        d = self._dev(hologram, precision)
        out = d.new_empty((cfg.num_planes,) + tuple(d.shape))
        L.check(self.lib.holo_inverse_propagate(self.h, d.data_ptr(), out.data_ptr(), C.byref(_wave(cfg)),
                                                C.byref(_prop(opt)), _NP[precision][0]))
        r = out.cpu().numpy()
        return [r[l] for l in range(r.shape[0])]

    def intensity(self, u: np.ndarray, precision: str = "f64") -> np.ndarray:
        d = self._dev(u, precision)
        torch = _torch()
        out = torch.empty(d.shape, dtype=torch.float32 if precision == "f32" else torch.float64, device=d.device)
        L.check(self.lib.holo_intensity(self.h, d.data_ptr(), out.data_ptr(), d.numel(), _NP[precision][0]))
        return out.cpu().numpy()


class Optimizer:
    """OptimState + optimizer_step (optimizer.hpp:37-58) on a context's resident
    scene: device moments, updates in place in HBM."""

    def __init__(self, ctx: "Context"):
        self.ctx = ctx
        h = C.c_void_p()
        L.check(ctx.lib.holo_optim_create(ctx.h, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            L.check(self.ctx.lib.holo_optim_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, grads: dict, cfg: Optional[OptimizerConfig] = None) -> bool:
        """One update from device f64 gradient tensors (as total_loss returns);
        False (and a counted skip) when a gradient is non-finite."""
        g = L.SceneGrads()
        for k in L.GRAD_FIELDS:
            if k != "mu_screen":
                setattr(g, k, grads[k].data_ptr())
        applied = C.c_int(0)
        L.check(self.ctx.lib.holo_optim_step(self.ctx.h, self.h, C.byref(g), C.byref(_optim_cfg(cfg)),
                                             C.byref(applied)))
        return bool(applied.value)

    def counts(self):
        s, k = C.c_longlong(), C.c_longlong()
        L.check(self.ctx.lib.holo_optim_counts(self.h, C.byref(s), C.byref(k)))
        return int(s.value), int(k.value)


_DEFAULT: dict = {}


def _scene_arrays(scene: GaussianScene):
    n = scene.size()
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
            (scene.positions, scene.rotations, scene.log_scales, scene.amplitudes, scene.opacity_logits,
             scene.phases, scene.plane_logits)]
    if [a.size for a in arrs] != [3 * n, 4 * n, 3 * n, 3 * n, n, 3 * n, n * scene.num_planes]:
        raise HoloError("config", "scene arrays have inconsistent sizes")
    s = L.SceneArrays()
    s.n, s.num_planes = n, int(scene.num_planes)
    for name, a in zip(("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases",
                        "plane_logits"), arrs):
        setattr(s, name, a.ctypes.data)
    return s, arrs


def mesh_layout(world: int, rank: int, plane_split: int, num_planes: int, num_views: int = 1,
                channels: int = 3) -> L.Mesh:
    """holo_mesh_layout: pure host arithmetic of the (view groups x plane split) mesh."""
    m = L.Mesh()
    L.check(L.lib().holo_mesh_layout(int(world), int(rank), int(plane_split), int(num_planes), int(num_views),
                                     int(channels), C.byref(m)))
    return m


def gloo_allreduce(group=None):
    """An all-reduce callback for Group(transport=callback) that sums through a
    torch.distributed process group on host memory (gloo): the transport the
    world-2/4 tests use when every rank shares one GPU (NCCL refuses two ranks on
    one device).  Blocking; production groups use NCCL."""
    torch = _torch()
    import torch.distributed as dist

    def fn(user, buf, count, stream):
        try:
            torch.cuda.ExternalStream(int(stream or 0)).synchronize()
            dev = torch.as_tensor(_CudaArray(int(buf), (int(count),), "<f4"), device="cuda")
            host = dev.cpu()
            dist.all_reduce(host, group=group)
            dev.copy_(host)
            torch.cuda.synchronize()
            return 0
        except Exception as e:  # noqa: BLE001 - reported as a status code to the library
            print(f"gloo_allreduce: {e!r}")
            return 1

    return fn


class Group:
    """holo_group (include/holo_cuda.h): this process's ranks of a multi-GPU render
    -- plane sharding (C3), view sharding (C4) or planes x views (C5).

    ``ctx``: this rank's Context (one process per GPU).  ``plane_split``: ranks per
    plane group (default: world, planes only; 1: views only).  Transport: NCCL from
    ``unique_id`` (rank 0's ``Group.unique_id()``, shared by the caller), or
    ``allreduce`` = a Python callable (see gloo_allreduce)."""

    def __init__(self, ctx: Context, world: int = 1, rank: int = 0, plane_split: Optional[int] = None,
                 unique_id: Optional[bytes] = None, allreduce=None):
        self.lib = L.lib()
        self.ctx, self.world, self.rank = ctx, int(world), int(rank)
        self.plane_split = int(world if plane_split is None else plane_split)
        h = C.c_void_p()
        self._cb = None
        if allreduce is not None:
            self._cb = L.ALLREDUCE_FN(allreduce)
            L.check(self.lib.holo_group_init_callback(ctx.h, self.world, self.rank, self.plane_split, self._cb, None,
                                                      C.byref(h)))
        else:
            uid = unique_id if unique_id is not None else (Group.unique_id() if self.world == 1 else None)
            if uid is None or len(uid) != L.GROUP_ID_BYTES:
                raise HoloError("usage", "Group: NCCL transport needs rank 0's 128-byte unique id")
            L.check(self.lib.holo_group_init_rank(ctx.h, bytes(uid), self.world, self.rank, self.plane_split,
                                                  C.byref(h)))
        self.h = h
        self._keep = []

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(L.GROUP_ID_BYTES)
        L.check(L.lib().holo_group_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch(cls, ctx: Context, plane_split: Optional[int] = None, group=None):
        """NCCL group over the ranks of a torch.distributed process group (the
        unique id is broadcast from rank 0 through it)."""
        import torch.distributed as dist

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        obj = [Group.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(ctx, world, rank, plane_split, unique_id=obj[0])

    def close(self):
        if getattr(self, "h", None):
            L.check(self.lib.holo_group_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def mesh(self, num_planes: int, num_views: int = 1, channels: int = 3) -> L.Mesh:
        m = L.Mesh()
        L.check(self.lib.holo_group_mesh(self.h, 0, int(num_planes), int(num_views), int(channels), C.byref(m)))
        return m

    def set_lanes(self, lanes: int) -> None:
        """Frames in flight on this rank (each lane: own stream and scene copy)."""
        L.check(self.lib.holo_group_set_lanes(self.h, int(lanes)))

    def upload_scene(self, scene: GaussianScene) -> None:
        """The full scene; a plane-sharded rank keeps its planes' Gaussians (on the device)."""
        s, arrs = _scene_arrays(scene)
        L.check(self.lib.holo_group_upload_scene(self.h, C.byref(s)))
        self._keep = arrs

    def render(self, cams: Sequence[CameraView], cfg: WaveConfig, settings: Optional[RenderSettings] = None,
               prop: Optional[PropagationOptions] = None, outputs: int = L.OUT_HOLOGRAM | L.OUT_INTENSITY,
               flags: int = 0, view_outputs: Optional[dict] = None) -> List[L.FrameInfo]:
        """Render this rank's share of the views ``cams``.  view_outputs: {view:
        (hologram, replayed, intensities)} caller device tensors (None members: the
        context's buffers).  Returns the FrameInfo of every view (zeros for views
        rendered elsewhere, and for asynchronous frames)."""
        V = len(cams)
        cam_arr = (L.Camera * V)(*[_camera(c) for c in cams])
        infos = (L.FrameInfo * V)()
        outs = None
        if view_outputs:
            outs = (L.ViewOutputs * V)()
            for v, (hh, rr, ii) in view_outputs.items():
                outs[v].hologram = hh.data_ptr() if hh is not None else None
                outs[v].replayed = rr.data_ptr() if rr is not None else None
                outs[v].intensities = ii.data_ptr() if ii is not None else None
        L.check(self.lib.holo_group_render(self.h, cam_arr, V, C.byref(_wave(cfg)), C.byref(_settings(settings)),
                                           C.byref(_prop(prop)), int(outputs), int(flags), outs, infos))
        return list(infos)

    def synchronize(self) -> None:
        L.check(self.lib.holo_group_synchronize(self.h))

    def set_async(self, on: bool = True) -> None:
        L.check(self.lib.holo_group_set_async(self.h, int(on)))

    def frame_status(self) -> None:
        L.check(self.lib.holo_group_frame_status(self.h))

    def join(self, stream: int) -> None:
        """Make CUDA stream `stream` wait for all of this rank's enqueued work."""
        L.check(self.lib.holo_group_join(self.h, 0, C.c_void_p(int(stream) or None)))

    def launch_count(self) -> int:
        return int(self.lib.holo_group_launch_count(self.h))


def default_context(device: int = 0) -> Context:
    ctx = _DEFAULT.get(device)
    if ctx is None:
        ctx = Context(device)
        _DEFAULT[device] = ctx
    return ctx


# ------------------------------------------------------------------ reference-shaped functions

def _collect_raster(ctx: Context, scene: GaussianScene, cfg: WaveConfig, C_: int, info: L.FrameInfo,
                    want_aux: bool = True) -> RasterForward:
    Ln, H, W = cfg.num_planes, cfg.ny, cfg.nx
    N = scene.size()
    layers = ctx.download(L.BUF_LAYERS, np.complex64, (Ln, C_, H, W)).astype(np.complex128)
    t_final = n_contrib = None
    if want_aux:
        t_final = ctx.download(L.BUF_T_FINAL, np.float32, (Ln, H, W)).astype(np.float64)
        n_contrib = ctx.download(L.BUF_N_CONTRIB, np.int32, (Ln, H, W))
    E = int(info.num_entries)
    B = Ln * info.tiles_x * info.tiles_y
    bucket_start = ctx.download(L.BUF_BUCKET_START, np.uint32, (B + 1,))
    gidx = ctx.download(L.BUF_ENTRY_GIDX, np.int32, (E,))
    depth = ctx.download(L.BUF_ENTRY_DEPTH, np.float64, (E,))
    entries = np.zeros(E, dtype=[("bucket", np.int32), ("gidx", np.int32), ("depth", np.float64)])
    entries["bucket"] = np.repeat(np.arange(B, dtype=np.int32), np.diff(bucket_start.astype(np.int64)))
    entries["gidx"] = gidx
    entries["depth"] = depth
    proj = ctx.download(L.BUF_PROJECTED, np.uint8, (N * C.sizeof(L.Projected),))
    pa = np.frombuffer(proj.tobytes(), dtype=np.dtype([(n, "<i4") if t in (C.c_int32,) else
                                                       (n, "<f8", (3,)) if n in ("amp", "phase") else (n, "<f8")
                                                       for n, t in L.Projected._fields_]))
    projected = {k: pa[k].copy() for k in pa.dtype.names if k != "pad_"}
    rho = ctx.download(L.BUF_RHO, np.float64, (N, Ln))
    touched = ctx.download(L.BUF_TOUCHED, np.uint8, (N,))
    return RasterForward(layers=[layers[l] for l in range(Ln)], t_final=t_final, n_contrib=n_contrib,
                         projected=projected, rho=rho, touched=touched, entries=entries, bucket_start=bucket_start,
                         tiles_x=int(info.tiles_x), tiles_y=int(info.tiles_y))


def _check_shapes(scene: GaussianScene, cam: CameraView, cfg: WaveConfig) -> None:
    scene.validate()
    cam.validate()
    cfg.validate()
    if scene.num_planes != cfg.num_planes:
        raise HoloError("config", "scene plane count does not match the wave config")
    if cam.width != cfg.nx or cam.height != cfg.ny:
        raise HoloError("config", "camera resolution must match the hologram grid")


def raster_forward(scene: GaussianScene, cam: CameraView, cfg: WaveConfig,
                   settings: Optional[RenderSettings] = None, ctx: Optional[Context] = None) -> RasterForward:
    """rasterizer.cpp:139-263 on the GPU.  Layers carry cfg.channels() channels when
    cfg has fewer than 3 wavelengths (C1 adapter), else the reference's 3."""
    _check_shapes(scene, cam, cfg)
    ctx = ctx or default_context()
    ctx.upload_scene(scene)
    C_ = min(cfg.channels(), 3)
    cfg3 = cfg if cfg.channels() <= 3 else WaveConfig(cfg.nx, cfg.ny, cfg.pitch, list(cfg.wavelengths)[:3],
                                                      cfg.distance, cfg.volume_depth, cfg.num_planes)
    info = ctx.render(cam, cfg3, settings, None,
                      outputs=L.OUT_LAYERS | L.OUT_AUX | L.OUT_LISTS | L.OUT_PROJECTED)
    return _collect_raster(ctx, scene, cfg3, C_, info)


def brute_force_forward(scene: GaussianScene, cam: CameraView, cfg: WaveConfig,
                        settings: Optional[RenderSettings] = None, ctx: Optional[Context] = None) -> List[np.ndarray]:
    """holo::brute_force_forward (rasterizer.cpp:265-315) on the GPU: every valid
    Gaussian of a plane at every pixel in the global (depth, index) order, no
    tiles, no radius culling, no early termination.  Layers [C, H, W] per plane."""
    _check_shapes(scene, cam, cfg)
    ctx = ctx or default_context()
    ctx.upload_scene(scene)
    L.check(ctx.lib.holo_brute_force_forward(ctx.h, C.byref(_camera(cam)), C.byref(_wave(cfg)),
                                             C.byref(_settings(settings))))
    lay = ctx.download(L.BUF_LAYERS, np.complex64, (cfg.num_planes, cfg.channels(), cfg.ny, cfg.nx))
    return [lay[l].astype(np.complex128) for l in range(cfg.num_planes)]


def pipeline_forward(scene: GaussianScene, cam: CameraView, cfg: WaveConfig,
                     opt: Optional[PipelineOptions] = None, ctx: Optional[Context] = None,
                     raster: bool = True, replayed: bool = True) -> PipelineForward:
    """pipeline.cpp:20-29: raster -> forward_record -> inverse_propagate -> intensity."""
    _check_shapes(scene, cam, cfg)
    if cfg.channels() > 3:
        raise HoloError("config", "propagate: field does not match the configured grid")
    opt = opt or PipelineOptions()
    ctx = ctx or default_context()
    ctx.upload_scene(scene)
    outs = L.OUT_HOLOGRAM | L.OUT_INTENSITY
    if replayed:
        outs |= L.OUT_REPLAYED
    if raster:
        outs |= L.OUT_LAYERS | L.OUT_AUX | L.OUT_LISTS | L.OUT_PROJECTED
    info = ctx.render(cam, cfg, opt.raster, opt.prop, outputs=outs)
    Cn, Ln, H, W = cfg.channels(), cfg.num_planes, cfg.ny, cfg.nx
    holo = ctx.download(L.BUF_HOLOGRAM, np.complex64, (Cn, H, W)).astype(np.complex128)
    ints = ctx.download(L.BUF_INTENSITY, np.float32, (Ln, Cn, H, W)).astype(np.float64)
    rep = None
    if replayed:
        r = ctx.download(L.BUF_REPLAYED, np.complex64, (Ln, Cn, H, W)).astype(np.complex128)
        rep = [r[l] for l in range(Ln)]
    ras = _collect_raster(ctx, scene, cfg, Cn, info) if raster else None
    return PipelineForward(raster=ras, hologram=holo, replayed=rep, intensities=[ints[l] for l in range(Ln)])


def raster_backward(scene: GaussianScene, cam: CameraView, cfg: WaveConfig, settings: Optional[RenderSettings],
                    grad_layers, ctx: Optional[Context] = None) -> dict:
    """rasterizer.hpp:79-81: scene gradients for dL/d(layers) [L, C, H, W] (numpy);
    renders the raster forward first, as the reference's caller does."""
    torch = _torch()
    _check_shapes(scene, cam, cfg)
    ctx = ctx or default_context()
    ctx.upload_scene(scene)
    ctx.render(cam, cfg, settings, None, outputs=L.OUT_LAYERS | L.OUT_AUX)
    gl = torch.from_numpy(np.ascontiguousarray(grad_layers, dtype=np.complex64)).to(f"cuda:{ctx.device}")
    out = ctx.raster_backward(cam, cfg, settings, gl, scene.size())
    return {k: v.cpu().numpy() for k, v in out.items()}


def pipeline_backward(scene: GaussianScene, cam: CameraView, cfg: WaveConfig, opt: Optional[PipelineOptions],
                      grad_intensities, ctx: Optional[Context] = None):
    """The gradient branch of total_loss (pipeline.cpp:63-80) for dL/dI [L, C, H, W]
    (numpy): returns (scene gradients, grad_layers, grad_hologram) as numpy."""
    torch = _torch()
    _check_shapes(scene, cam, cfg)
    opt = opt or PipelineOptions()
    ctx = ctx or default_context()
    ctx.upload_scene(scene)
    ctx.render(cam, cfg, opt.raster, opt.prop, outputs=L.OUT_HOLOGRAM | L.OUT_REPLAYED | L.OUT_AUX)
    gi = torch.from_numpy(np.ascontiguousarray(grad_intensities, dtype=np.float32)).to(f"cuda:{ctx.device}")
    out, gl, gh = ctx.pipeline_backward(cam, cfg, opt.raster, opt.prop, gi, scene.size())
    return ({k: v.cpu().numpy() for k, v in out.items()}, gl.cpu().numpy().astype(np.complex128),
            gh.cpu().numpy().astype(np.complex128))


def losses(I, I_gt, masks, opt: Optional[PipelineOptions] = None, ctx: Optional[Context] = None):
    """losses.hpp on numpy stacks [L, C, H, W] (masks [L, H, W] or None for plain
    MSE): returns (LossBreakdown, dL/dI as numpy)."""
    torch = _torch()
    ctx = ctx or default_context()
    dev = f"cuda:{ctx.device}"
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)  # noqa: E731
    b, g = ctx.losses(t(I), t(I_gt), t(masks) if masks is not None else None, opt)
    return b, g.cpu().numpy()


def total_loss(scene: GaussianScene, cam: CameraView, cfg: WaveConfig, images, masks,
               opt: Optional[PipelineOptions] = None, want_grads: bool = True, ctx: Optional[Context] = None):
    """pipeline.hpp:54-56 (FocalStackTarget given as images [L, C, H, W] and masks
    [L, H, W]): returns (LossBreakdown, gradients as numpy or None)."""
    torch = _torch()
    _check_shapes(scene, cam, cfg)
    ctx = ctx or default_context()
    ctx.upload_scene(scene)
    dev = f"cuda:{ctx.device}"
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)  # noqa: E731
    b, out = ctx.total_loss(cam, cfg, t(images), t(masks) if masks is not None else None, opt,
                            scene.size() if want_grads else None)
    return b, ({k: v.cpu().numpy() for k, v in out.items()} if out is not None else None)


def _phase_inputs(P, cfg: WaveConfig, ctx: "Context"):
    torch = _torch()
    P = np.ascontiguousarray(P, dtype=np.complex128)
    if P.ndim != 3 or P.shape != (cfg.channels(), cfg.ny, cfg.nx):
        raise HoloError("config", "hologram shape does not match the wave config")  # phase_only.cpp:24-25
    return P, torch.from_numpy(P).to(f"cuda:{ctx.device}")


def phase_only_loss(P, theta, cfg: WaveConfig, opt: Optional[PhaseOnlyOptions] = None, want_grad: bool = False,
                    ctx: Optional[Context] = None):
    """phase_only.hpp:39-40 on numpy arrays ([C, H, W]): the loss, and with
    want_grad also d loss / d theta."""
    torch = _torch()
    ctx = ctx or default_context()
    P, dP = _phase_inputs(P, cfg, ctx)
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    if theta.size != P.size:
        raise HoloError("config", "phase vector does not match the hologram shape")
    dt = torch.from_numpy(theta.reshape(P.shape)).to(dP.device)
    g = torch.empty_like(dt) if want_grad else None
    loss = ctx.phase_only_loss(dP, dt, cfg, opt, g)
    return (loss, g.cpu().numpy()) if want_grad else loss


def convert_phase_only(P, cfg: WaveConfig, iters: int = 1000, lr: float = 0.02,
                       opt: Optional[PhaseOnlyOptions] = None, ctx: Optional[Context] = None) -> PhaseOnlyResult:
    """phase_only.hpp:49-50.  The starting phase arg(P) is taken on the host (the
    reference's std::arg, bit for bit); the iterations run on the GPU."""
    torch = _torch()
    ctx = ctx or default_context()
    P, dP = _phase_inputs(P, cfg, ctx)
    theta0 = torch.from_numpy(np.ascontiguousarray(np.angle(P))).to(dP.device)
    out, trace = ctx.convert_phase_only(dP, cfg, iters, lr, opt, theta0)
    return PhaseOnlyResult(hologram=PhaseOnlyHologram(phase=out.cpu().numpy()), trace=trace)


def phase_gradient_oracle(P, theta, cfg: WaveConfig, indices: Optional[Sequence[int]] = None, fd_step: float = 1e-5,
                          opt: Optional[PhaseOnlyOptions] = None, ctx: Optional[Context] = None) -> np.ndarray:
    """phase_only.hpp:56-62: central differences of the matching loss at the sampled
    entries (all when indices is empty), each loss evaluated on the GPU."""
    torch = _torch()
    if cfg.num_planes < 1:
        raise HoloError("config", "oracle needs at least one depth plane")
    if cfg.nx > 64 or cfg.ny > 64:
        raise HoloError("config", "oracle is limited to grids up to 64x64")
    ctx = ctx or default_context()
    P, dP = _phase_inputs(P, cfg, ctx)
    theta = np.ascontiguousarray(theta, dtype=np.float64).ravel()
    if theta.size != P.size:
        raise HoloError("config", "phase vector does not match the hologram shape")
    if not fd_step > 0.0:
        raise HoloError("config", "difference step must be positive")
    idx = list(range(theta.size)) if not indices else [int(i) for i in indices]
    g = np.zeros(theta.size)
    probe = theta.copy()
    for i in idx:
        if i < 0 or i >= theta.size:
            raise HoloError("config", "sampled phase index out of range")
        vals = []
        for v in (theta[i] + fd_step, theta[i] - fd_step):
            probe[i] = v
            vals.append(ctx.phase_only_loss(dP, torch.from_numpy(probe.reshape(P.shape)).to(dP.device), cfg, opt))
        probe[i] = theta[i]
        g[i] = (vals[0] - vals[1]) / (2.0 * fd_step)
    return g


def propagate(u, cfg: WaveConfig, z: float, opt: Optional[PropagationOptions] = None, precision: str = "f64"):
    return default_context().propagate(u, cfg, z, opt, precision)


def forward_record(layers, cfg: WaveConfig, opt: Optional[PropagationOptions] = None, precision: str = "f64"):
    return default_context().forward_record(layers, cfg, opt, precision)


def inverse_propagate(hologram, cfg: WaveConfig, opt: Optional[PropagationOptions] = None, precision: str = "f64"):
    return default_context().inverse_propagate(hologram, cfg, opt, precision)


def transfer_function(cfg: WaveConfig, z: float, opt: Optional[PropagationOptions] = None, precision: str = "f64"):
    return default_context().transfer_function(cfg, z, opt, precision)


def fft2(data, precision: str = "f64"):
    return default_context().fft2(data, False, precision)


def ifft2(data, precision: str = "f64"):
    return default_context().fft2(data, True, precision)


def intensity(u, precision: str = "f64"):
    return default_context().intensity(u, precision)
