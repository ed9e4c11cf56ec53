"""ctypes front end to the CPU oracles.

TEST INFRASTRUCTURE.  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this module; the
product package never does.

Two backends expose the same Python API:

* ``Oracle("restate")`` -- oracle/_build/libholo_oracle.so, the plain-C
  restatement of the reference forward path (oracle/holo_oracle.c);
* ``Oracle("ref")`` -- oracle/_ref/libref_capi.so, the reference's own C++
  sources (/root/reference/proj/src) compiled in place against the shims in
  oracle/shim (see oracle/Makefile).  Present only where that build ran.

Arguments are duck-typed on the reference's type names (WaveConfig,
CameraView, GaussianScene, RenderSettings, PropagationOptions): any object with
the same attribute names works, so the product's dataclasses and the plain
namespaces used by the fixture generator both pass.  Fields are numpy
complex128 arrays shaped [C, H, W] (per plane: [L, C, H, W]), the reference's
planar layout (proj/include/holo/field.hpp:9-21).
"""
from __future__ import annotations

import ctypes as C
import os
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MAX_CH = 16


class _Wave(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("pitch", C.c_double), ("channels", C.c_int),
                ("wavelengths", C.c_double * MAX_CH), ("distance", C.c_double), ("volume_depth", C.c_double),
                ("num_planes", C.c_int)]


class _Camera(C.Structure):
    _fields_ = [("pose", C.c_double * 6), ("focal_px", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int), ("height", C.c_int)]


class _Settings(C.Structure):
    _fields_ = [("near_clip", C.c_double), ("dilation", C.c_double), ("plane_eps", C.c_double),
                ("term_eps", C.c_double), ("alpha_floor", C.c_double), ("alpha_clamp", C.c_double),
                ("radius_form_cap", C.c_double), ("ste_tau", C.c_double), ("soft_assignment", C.c_int),
                ("soft_tau", C.c_double), ("tile", C.c_int)]


class _Prop(C.Structure):
    _fields_ = [("pad2x", C.c_int), ("local_band_limit", C.c_int)]


_dp = C.POINTER(C.c_double)


class _Scene(C.Structure):
    _fields_ = [("n", C.c_size_t), ("num_planes", C.c_int), ("positions", _dp), ("rotations", _dp),
                ("log_scales", _dp), ("amplitudes", _dp), ("opacity_logits", _dp), ("phases", _dp),
                ("plane_logits", _dp)]


class _Projected(C.Structure):
    _fields_ = [("valid", C.c_int), ("n", C.c_int), ("mu_x", C.c_double), ("mu_y", C.c_double),
                ("inv00", C.c_double), ("inv01", C.c_double), ("inv11", C.c_double), ("radius", C.c_double),
                ("xc", C.c_double), ("yc", C.c_double), ("zc", C.c_double), ("alpha_sig", C.c_double),
                ("amp", C.c_double * 3), ("phase", C.c_double * 3), ("plane", C.c_int)]


class _Raster(C.Structure):
    _fields_ = [("L", C.c_int), ("w", C.c_int), ("h", C.c_int), ("tiles_x", C.c_int), ("tiles_y", C.c_int),
                ("num_entries", C.c_size_t), ("layers", _dp), ("t_final", _dp),
                ("n_contrib", C.POINTER(C.c_int32)), ("projected", C.POINTER(_Projected)), ("rho", _dp),
                ("touched", C.POINTER(C.c_uint8)), ("entry_bucket", C.POINTER(C.c_int32)),
                ("entry_gidx", C.POINTER(C.c_int32)), ("entry_depth", _dp),
                ("bucket_start", C.POINTER(C.c_uint32))]


class _Grads(C.Structure):
    _fields_ = [(k, _dp) for k in ("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases",
                                   "plane_logits", "mu_screen")]


class OracleError(RuntimeError):
    """Mirror of holo::HoloError (common.hpp:76-79): ``kind`` in config/io/usage/numeric."""

    KINDS = {1: "config", 2: "io", 3: "usage", 4: "numeric"}

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.kind = self.KINDS.get(code, "numeric")


DEFAULT_SETTINGS = dict(near_clip=0.0, dilation=0.3, plane_eps=0.5, term_eps=1e-4, alpha_floor=1.0 / 255.0,
                        alpha_clamp=0.999, radius_form_cap=0.0, ste_tau=1e-3, soft_assignment=False, soft_tau=1.0,
                        tile=16)


def _get(obj, name, default=None):
    if obj is None:
        return default
    if isinstance(obj, dict):
        return obj.get(name, default)
    return getattr(obj, name, default)


def _wave(w) -> _Wave:
    wl = list(_get(w, "wavelengths"))
    s = _Wave()
    s.nx, s.ny = int(_get(w, "nx")), int(_get(w, "ny"))
    s.pitch = float(_get(w, "pitch", 3.74e-6))
    s.channels = len(wl)
    for i, v in enumerate(wl):
        s.wavelengths[i] = float(v)
    s.distance = float(_get(w, "distance", 2e-3))
    s.volume_depth = float(_get(w, "volume_depth", 4e-3))
    s.num_planes = int(_get(w, "num_planes"))
    return s


def _camera(c) -> _Camera:
    s = _Camera()
    pose = list(_get(c, "pose", [0.0] * 6))
    for i in range(6):
        s.pose[i] = float(pose[i])
    s.focal_px = float(_get(c, "focal_px", 150.0))
    s.cx, s.cy = float(_get(c, "cx", -1.0)), float(_get(c, "cy", -1.0))
    s.width, s.height = int(_get(c, "width")), int(_get(c, "height"))
    return s


def _settings(st) -> _Settings:
    s = _Settings()
    for k, d in DEFAULT_SETTINGS.items():
        v = _get(st, k, d)
        setattr(s, k, int(v) if k in ("soft_assignment", "tile") else float(v))
    return s


def _prop(p) -> _Prop:
    s = _Prop()
    s.pad2x = int(bool(_get(p, "pad2x", False)))
    s.local_band_limit = int(bool(_get(p, "local_band_limit", False)))
    return s


def _f64(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64).ravel()
    if n is not None and a.size != n:
        raise OracleError(1, "scene arrays have inconsistent sizes")
    return a


class _SceneArgs:
    """Keeps the contiguous f64 arrays alive for the duration of a call."""

    def __init__(self, sc, copy=False):
        n = len(np.asarray(_get(sc, "opacity_logits")).ravel())
        L = int(_get(sc, "num_planes"))
        self.arrays = [_f64(_get(sc, "positions"), 3 * n), _f64(_get(sc, "rotations"), 4 * n),
                       _f64(_get(sc, "log_scales"), 3 * n), _f64(_get(sc, "amplitudes"), 3 * n),
                       _f64(_get(sc, "opacity_logits"), n), _f64(_get(sc, "phases"), 3 * n),
                       _f64(_get(sc, "plane_logits"), n * L)]
        if copy:  # callee writes the arrays: never alias the caller's scene
            self.arrays = [a.copy() for a in self.arrays]
        self.s = _Scene()
        self.s.n, self.s.num_planes = n, L
        for name, arr in zip(["positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases",
                              "plane_logits"], self.arrays):
            setattr(self.s, name, arr.ctypes.data_as(_dp))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


class Oracle:
    def __init__(self, kind: str = "restate"):
        self.kind = kind
        if kind == "restate":
            path = os.path.join(HERE, "_build", "libholo_oracle.so")
            pre = "ho_"
        elif kind == "ref":
            path = os.path.join(HERE, "_ref", "libref_capi.so")
            pre = "ref_"
        else:
            raise ValueError(kind)
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle backend {kind!r} not built: {path} (run make -C oracle)")
        self.lib = C.CDLL(path)
        self.pre = pre
        L = self.lib
        getattr(L, pre + "last_error").restype = C.c_char_p
        self._free = getattr(L, pre + "raster_free")

    @staticmethod
    def available(kind: str) -> bool:
        sub = {"restate": ("_build", "libholo_oracle.so"), "ref": ("_ref", "libref_capi.so")}[kind]
        return os.path.exists(os.path.join(HERE, *sub))

    def _fn(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._fn("last_error")().decode())

    # ----------------------------------------------------------- small pieces
    def covariance_3d(self, quat, log_scales):
        """covariance_3d (scene.cpp:125-130), restatement only; returns 3x3."""
        q = np.ascontiguousarray(quat, dtype=np.float64)
        s = np.ascontiguousarray(log_scales, dtype=np.float64)
        out = np.zeros(9)
        self.lib.ho_covariance_3d(_ptr(q), _ptr(s), _ptr(out))
        return out.reshape(3, 3)

    def ste_argmax(self, logits):
        a = np.ascontiguousarray(logits, dtype=np.float64)
        return int(self.lib.ho_ste_argmax(_ptr(a), C.c_int(a.size)))

    def plane_positions(self, wave):
        wv = _wave(wave)
        z = np.zeros(wv.num_planes)
        self._check(self.lib.ho_plane_positions(C.byref(wv), _ptr(z)))
        return z

    # ---------------------------------------------------------------- raster
    def _unpack_raster(self, r: _Raster, N: int):
        L, h, w = r.L, r.h, r.w
        P = w * h
        E = r.num_entries
        B = L * r.tiles_x * r.tiles_y

        def arr(ptr, n, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)

        layers = arr(r.layers, L * 3 * P * 2, np.float64).view(np.complex128).reshape(L, 3, h, w)
        projected = {name: np.zeros(0) for name, _ in _Projected._fields_}
        if N:
            proj = np.ctypeslib.as_array(r.projected, shape=(N,))
            projected = {k: np.array(proj[k], copy=True) for k in proj.dtype.names}
        out = SimpleNamespace(
            layers=layers,
            t_final=arr(r.t_final, L * P, np.float64).reshape(L, h, w),
            n_contrib=arr(r.n_contrib, L * P, np.int32).reshape(L, h, w),
            touched=arr(r.touched, N, np.uint8),
            rho=arr(r.rho, N * L, np.float64).reshape(N, L),
            entry_bucket=arr(r.entry_bucket, E, np.int32),
            entry_gidx=arr(r.entry_gidx, E, np.int32),
            entry_depth=arr(r.entry_depth, E, np.float64),
            bucket_start=arr(r.bucket_start, B + 1, np.uint32),
            tiles_x=r.tiles_x, tiles_y=r.tiles_y, projected=projected)
        self._free(C.byref(r))
        return out

    def raster_forward(self, scene, cam, wave, settings=None):
        sa = _SceneArgs(scene)
        r = _Raster()
        self._check(self._fn("raster_forward")(C.byref(sa.s), C.byref(_camera(cam)), C.byref(_wave(wave)),
                                               C.byref(_settings(settings)), C.byref(r)))
        return self._unpack_raster(r, sa.s.n)

    def brute_force_forward(self, scene, cam, wave, settings=None):
        sa = _SceneArgs(scene)
        wv = _wave(wave)
        out = np.zeros((wv.num_planes, 3, wv.ny, wv.nx), dtype=np.complex128)
        self._check(self._fn("brute_force_forward")(C.byref(sa.s), C.byref(_camera(cam)), C.byref(wv),
                                                    C.byref(_settings(settings)), _ptr(out)))
        return out

    # ----------------------------------------------------------- propagation
    def fft2(self, field, inverse=False):
        a = _c128(field).copy()
        h, w = a.shape[-2:]
        for plane in a.reshape(-1, h, w):
            if self.kind == "ref":
                self._check(self.lib.ref_fft2(_ptr(plane), w, h, int(inverse)))
            else:
                (self.lib.ho_ifft2 if inverse else self.lib.ho_fft2)(_ptr(plane), w, h)
        return a

    def transfer_function(self, wave, z, prop=None):
        wv = _wave(wave)
        pp = _prop(prop)
        f = 2 if pp.pad2x else 1
        out = np.zeros((wv.channels, wv.ny * f, wv.nx * f), dtype=np.complex128)
        self._check(self._fn("transfer_function")(C.byref(wv), C.c_double(z), C.byref(pp), _ptr(out)))
        return out

    def propagate(self, field, wave, z, prop=None):
        a = _c128(field)
        c, h, w = a.shape
        out = np.empty_like(a)
        self._check(self._fn("propagate")(_ptr(a), w, h, c, C.byref(_wave(wave)), C.c_double(z),
                                          C.byref(_prop(prop)), _ptr(out)))
        return out

    def forward_record(self, layers, wave, prop=None):
        a = _c128(layers)
        L, c, h, w = a.shape
        out = np.empty((c, h, w), dtype=np.complex128)
        if self.kind == "ref":
            rc = self.lib.ref_forward_record(_ptr(a), L, c, C.byref(_wave(wave)), C.byref(_prop(prop)), _ptr(out))
        else:
            rc = self.lib.ho_forward_record(_ptr(a), L, C.byref(_wave(wave)), C.byref(_prop(prop)), _ptr(out))
        self._check(rc)
        return out

    def inverse_propagate(self, holo, wave, prop=None):
        a = _c128(holo)
        c, h, w = a.shape
        wv = _wave(wave)
        out = np.empty((wv.num_planes, c, h, w), dtype=np.complex128)
        if self.kind == "ref":
            rc = self.lib.ref_inverse_propagate(_ptr(a), c, C.byref(wv), C.byref(_prop(prop)), _ptr(out))
        else:
            rc = self.lib.ho_inverse_propagate(_ptr(a), C.byref(wv), C.byref(_prop(prop)), _ptr(out))
        self._check(rc)
        return out

    # -------------------------------------------------------------- pipeline
    def pipeline_forward(self, scene, cam, wave, settings=None, prop=None, raster=True, replayed=True):
        """holo::pipeline_forward (pipeline.cpp:20-29).  Returns a namespace with
        hologram [C,H,W], replayed [L,C,H,W], intensities [L,C,H,W], raster
        (RasterForward fields) and stage_seconds (raster, record, replay, intensity)."""
        sa = _SceneArgs(scene)
        wv = _wave(wave)
        L, Cn, h, w = wv.num_planes, wv.channels, wv.ny, wv.nx
        holo = np.empty((Cn, h, w), dtype=np.complex128)
        rep = np.empty((L, Cn, h, w), dtype=np.complex128) if replayed else None
        ints = np.empty((L, Cn, h, w), dtype=np.float64)
        secs = np.zeros(4, dtype=np.float64)
        r = _Raster()
        rc = self._fn("pipeline_forward")(C.byref(sa.s), C.byref(_camera(cam)), C.byref(wv),
                                          C.byref(_settings(settings)), C.byref(_prop(prop)),
                                          C.byref(r) if raster else None, _ptr(holo), _ptr(rep), _ptr(ints),
                                          _ptr(secs))
        self._check(rc)
        ras = self._unpack_raster(r, sa.s.n) if raster else None
        return SimpleNamespace(hologram=holo, replayed=rep, intensities=ints, raster=ras, stage_seconds=secs)

    # -------------------------------------------------------------- gradients (reference build only)
    _GRAD_FIELDS = ("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases",
                    "plane_logits", "mu_screen")

    def _grads(self, n, L):
        shapes = {"positions": (n, 3), "rotations": (n, 4), "log_scales": (n, 3), "amplitudes": (n, 3),
                  "opacity_logits": (n,), "phases": (n, 3), "plane_logits": (n, L), "mu_screen": (n, 2)}
        arrays = {k: np.zeros(shapes[k]) for k in self._GRAD_FIELDS}
        g = _Grads()
        for k in self._GRAD_FIELDS:
            setattr(g, k, arrays[k].ctypes.data_as(_dp))
        return g, arrays

    def raster_backward(self, scene, cam, wave, settings, grad_layers):
        """holo::raster_backward (rasterizer.cpp:332-528) of raster_forward's
        output for dL/d(layers) [L,3,H,W]; returns a dict of scene gradients."""
        if self.kind != "ref":
            raise OracleError(3, "raster_backward needs the reference build")
        sa = _SceneArgs(scene)
        g, arrays = self._grads(sa.s.n, sa.s.num_planes)
        gl = _c128(grad_layers)
        self._check(self.lib.ref_raster_backward(C.byref(sa.s), C.byref(_camera(cam)), C.byref(_wave(wave)),
                                                 C.byref(_settings(settings)), _ptr(gl), C.byref(g)))
        return arrays

    def losses(self, I, I_gt, masks, lambda_ssim=0.005, plain=False):
        """The loss terms of total_loss (losses.cpp) on given stacks [L,C,H,W]:
        returns (recon, ssim, psnr [L], dL/dI [L,C,H,W])."""
        a = np.ascontiguousarray(I, dtype=np.float64)
        b = np.ascontiguousarray(I_gt, dtype=np.float64)
        L, Cn, H, W = a.shape
        m = np.ascontiguousarray(masks if masks is not None else np.zeros((L, H, W)), dtype=np.float64)
        out = np.zeros(2)
        ps = np.zeros(L)
        g = np.zeros_like(a)
        self._check(self.lib.ref_losses(_ptr(a), _ptr(b), _ptr(m), L, Cn, H, W, C.c_double(lambda_ssim), int(plain),
                                        _ptr(out), _ptr(ps), _ptr(g)))
        return out[0], out[1], ps, g

    def total_loss(self, scene, cam, wave, settings, prop, targets, masks, lambda_ssim=0.005, lambda_opacity=1e-4,
                   plain=False, grads=True):
        """holo::total_loss (pipeline.cpp:30-95): returns (breakdown dict, psnr [L], scene gradients or None)."""
        sa = _SceneArgs(scene)
        wv = _wave(wave)
        t = np.ascontiguousarray(targets, dtype=np.float64)
        m = np.ascontiguousarray(masks, dtype=np.float64)
        bd = np.zeros(5)
        ps = np.zeros(wv.num_planes)
        g, arrays = self._grads(sa.s.n, wv.num_planes)
        self._check(self.lib.ref_total_loss(C.byref(sa.s), C.byref(_camera(cam)), C.byref(wv),
                                            C.byref(_settings(settings)), C.byref(_prop(prop)),
                                            C.c_double(lambda_ssim), C.c_double(lambda_opacity), int(plain), _ptr(t),
                                            _ptr(m), _ptr(bd), _ptr(ps), C.byref(g) if grads else None))
        keys = ("recon", "ssim", "opacity", "total", "psnr_mean")
        return dict(zip(keys, bd.tolist())), ps, (arrays if grads else None)

    def optimizer_run(self, scene, grads_list, cfg, use_adam=False, schedule_total=20000):
        """holo::optimizer_step (optimizer.cpp:102-133) for each gradient dict of
        grads_list from fresh moments; returns (updated scene arrays, applied flags).
        cfg: [lr_pos, lr_rot, lr_logs, lr_amp, lr_phase, lr_opac, lr_plane, b1, b2, b3, eps, lr_floor]."""
        sa = _SceneArgs(scene, copy=True)
        order = ("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases", "plane_logits")
        packed = np.concatenate([np.concatenate([np.ravel(g[k]) for k in order]) for g in grads_list])
        applied = np.zeros(len(grads_list), dtype=np.int32)
        cv = np.ascontiguousarray(cfg, dtype=np.float64)
        self._check(self.lib.ref_optimizer_run(C.byref(sa.s), _ptr(packed), len(grads_list), _ptr(cv), int(use_adam),
                                               C.c_longlong(schedule_total),
                                               applied.ctypes.data_as(C.POINTER(C.c_int32))))
        names = order
        return {k: a.copy() for k, a in zip(names, sa.arrays)}, applied

    def phase_only_loss(self, P, theta, wave, lambda_ssim=1.0, prop=None, use_adam=False, grad=True):
        """holo::phase_only_loss (phase_only.cpp:104-111): (loss, d loss / d theta or None).
        prop defaults to PhaseOnlyOptions' pad2x = true."""
        a = _c128(P)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        pr = _prop(prop) if prop is not None else _prop({"pad2x": True})
        loss = C.c_double()
        g = np.zeros(a.shape) if grad else None
        self._check(self.lib.ref_phase_only_loss(_ptr(a), _ptr(th), C.byref(_wave(wave)), C.c_double(lambda_ssim),
                                                 C.byref(pr), int(use_adam), C.byref(loss),
                                                 _ptr(g) if grad else None))
        return loss.value, g

    def convert_phase_only(self, P, wave, iters=1000, lr=0.02, lambda_ssim=1.0, prop=None, use_adam=False):
        """holo::convert_phase_only (phase_only.cpp:113-160): (best phase [C,H,W], trace)."""
        a = _c128(P)
        pr = _prop(prop) if prop is not None else _prop({"pad2x": True})
        out = np.zeros(a.shape)
        trace = np.zeros(iters + 1)
        self._check(self.lib.ref_convert_phase_only(_ptr(a), C.byref(_wave(wave)), int(iters), C.c_double(lr),
                                                    C.c_double(lambda_ssim), C.byref(pr), int(use_adam), _ptr(out),
                                                    _ptr(trace)))
        return out, trace

    def pipeline_backward(self, scene, cam, wave, settings, prop, grad_intensities):
        """The gradient branch of holo::total_loss (pipeline.cpp:63-80) for
        dL/d(intensities) [L,C,H,W]: returns (scene gradients, grad_hologram,
        grad_layers)."""
        if self.kind != "ref":
            raise OracleError(3, "pipeline_backward needs the reference build")
        sa = _SceneArgs(scene)
        wv = _wave(wave)
        L, Cn, h, w = wv.num_planes, wv.channels, wv.ny, wv.nx
        g, arrays = self._grads(sa.s.n, L)
        gi = np.ascontiguousarray(grad_intensities, dtype=np.float64)
        gh = np.zeros((Cn, h, w), dtype=np.complex128)
        gl = np.zeros((L, Cn, h, w), dtype=np.complex128)
        self._check(self.lib.ref_pipeline_backward(C.byref(sa.s), C.byref(_camera(cam)), C.byref(wv),
                                                   C.byref(_settings(settings)), C.byref(_prop(prop)), _ptr(gi),
                                                   _ptr(gh), _ptr(gl), C.byref(g)))
        return arrays, gh, gl


def psnr(a, b) -> float:
    """holo::psnr (losses.cpp:113-132): min(99, 10 log10(1/MSE)), peak 1."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    mse = float(np.mean((a - b) ** 2))
    if mse <= 0.0:
        return 99.0
    return min(99.0, 10.0 * np.log10(1.0 / mse))


def rel_l2(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    den = float(np.linalg.norm(b.ravel()))
    num = float(np.linalg.norm((a - b).ravel()))
    return num / den if den > 0 else num
