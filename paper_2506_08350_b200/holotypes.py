"""Python mirror of the reference's render-path types (proj/include/holo/*.hpp).

Same names, fields, defaults and validation messages as the C++ structs so
callers and tests read like the reference:

* WaveConfig            wave_config.hpp:11-23, validate wave_config.cpp:5-16
* plane_positions       wave_config.cpp:18-30
* CameraView            camera.hpp:14-30, camera.cpp:5-27
* GaussianScene         scene.hpp:18-37, validate scene.cpp:19-32
* RenderSettings        rasterizer.hpp:12-28
* PropagationOptions    propagation.hpp:10-13
* PipelineOptions       pipeline.hpp:23-29 (render-relevant fields)
* RasterForward         rasterizer.hpp:63-73
* PipelineForward       pipeline.hpp:34-39
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._lib import HoloError


@dataclass
class WaveConfig:
    nx: int = 128
    ny: int = 128
    pitch: float = 3.74e-6
    wavelengths: Sequence[float] = (639e-9, 532e-9, 473e-9)
    distance: float = 2e-3
    volume_depth: float = 4e-3
    num_planes: int = 2

    def channels(self) -> int:
        return len(self.wavelengths)

    def validate(self) -> None:
        if self.nx <= 0 or self.ny <= 0:
            raise HoloError("config", "resolution must be positive")
        if self.pitch <= 0.0:
            raise HoloError("config", "pixel pitch must be positive")
        if len(self.wavelengths) == 0:
            raise HoloError("config", "at least one wavelength required")
        if any(l <= 0.0 for l in self.wavelengths):
            raise HoloError("config", "wavelengths must be positive")
        if self.distance <= 0.0:
            raise HoloError("config", "propagation distance must be positive")
        if self.volume_depth < 0.0:
            raise HoloError("config", "volume depth must be non-negative")
        if self.num_planes < 1:
            raise HoloError("config", "need at least one depth plane")
        if self.num_planes > 1 and self.volume_depth <= 0.0:
            raise HoloError("config", "multiple planes need a positive volume depth")


def plane_positions(cfg: WaveConfig) -> List[float]:
    """Z_l = d - (L-1)/2 dz + l dz, dz = depth / (L-1); [d] for L = 1 (wave_config.cpp:18-30)."""
    cfg.validate()
    L = cfg.num_planes
    if L == 1:
        return [float(cfg.distance)]
    dz = cfg.volume_depth / (L - 1)
    z0 = cfg.distance - 0.5 * (L - 1) * dz
    return [z0 + l * dz for l in range(L)]


def _mat3_mul(a, b):
    return [[(a[i][0] * b[0][j] + a[i][1] * b[1][j]) + a[i][2] * b[2][j] for j in range(3)] for i in range(3)]


@dataclass
class CameraView:
    pose: Sequence[float] = (0.0, 0.0, 0.0, 0.0, 0.0, 0.0)
    focal_px: float = 150.0
    cx: float = -1.0
    cy: float = -1.0
    width: int = 0
    height: int = 0

    def rot_cam_to_world(self) -> np.ndarray:
        """Rz(rz) Ry(ry) Rx(rx) (camera.cpp:5-14)."""
        cx_, sx_ = math.cos(self.pose[3]), math.sin(self.pose[3])
        cy_, sy_ = math.cos(self.pose[4]), math.sin(self.pose[4])
        cz_, sz_ = math.cos(self.pose[5]), math.sin(self.pose[5])
        rx = [[1, 0, 0], [0, cx_, -sx_], [0, sx_, cx_]]
        ry = [[cy_, 0, sy_], [0, 1, 0], [-sy_, 0, cy_]]
        rz = [[cz_, -sz_, 0], [sz_, cz_, 0], [0, 0, 1]]
        return np.array(_mat3_mul(_mat3_mul(rz, ry), rx), dtype=np.float64)

    def rot_world_to_cam(self) -> np.ndarray:
        return self.rot_cam_to_world().T.copy()

    def position(self) -> np.ndarray:
        return np.array(self.pose[:3], dtype=np.float64)

    def principal_x(self) -> float:
        return self.cx if self.cx >= 0.0 else self.width / 2.0

    def principal_y(self) -> float:
        return self.cy if self.cy >= 0.0 else self.height / 2.0

    def validate(self) -> None:
        if self.width <= 0 or self.height <= 0:
            raise HoloError("config", "camera resolution must be positive")
        if self.focal_px <= 0.0:
            raise HoloError("config", "focal length must be positive")
        if not all(math.isfinite(v) for v in self.pose):
            raise HoloError("config", "camera pose must be finite")


@dataclass
class GaussianScene:
    """Struct-of-arrays complex Gaussians; kChannels = 3 (scene.hpp:19)."""
    kChannels = 3
    num_planes: int = 1
    positions: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    rotations: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))
    log_scales: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    amplitudes: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    opacity_logits: np.ndarray = field(default_factory=lambda: np.zeros((0,)))
    phases: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    plane_logits: np.ndarray = field(default_factory=lambda: np.zeros((0, 1)))

    def size(self) -> int:
        return int(np.asarray(self.opacity_logits).size)

    def resize(self, n: int) -> None:
        """scene.cpp:8-17: identity rotations, everything else zero."""
        self.positions = np.zeros((n, 3))
        self.rotations = np.zeros((n, 4))
        self.rotations[:, 0] = 1.0
        self.log_scales = np.zeros((n, 3))
        self.amplitudes = np.zeros((n, 3))
        self.opacity_logits = np.zeros((n,))
        self.phases = np.zeros((n, 3))
        self.plane_logits = np.zeros((n, self.num_planes))

    def validate(self) -> None:
        n = self.size()
        if self.num_planes < 1:
            raise HoloError("config", "scene needs at least one plane")
        sizes = [np.asarray(a).size for a in (self.positions, self.rotations, self.log_scales, self.amplitudes,
                                              self.phases, self.plane_logits)]
        if sizes != [3 * n, 4 * n, 3 * n, 3 * n, 3 * n, n * self.num_planes]:
            raise HoloError("config", "scene arrays have inconsistent sizes")
        q = np.asarray(self.rotations, dtype=np.float64).reshape(n, 4)
        norm = np.sqrt(((q[:, 0] * q[:, 0] + q[:, 1] * q[:, 1]) + q[:, 2] * q[:, 2]) + q[:, 3] * q[:, 3])
        if n and not np.all(norm > 1e-8):
            raise HoloError("config", "degenerate quaternion in scene")
        if n and np.any(np.asarray(self.amplitudes) < 0.0):
            raise HoloError("config", "amplitudes must be non-negative")


@dataclass
class RenderSettings:
    near_clip: float = 0.0
    dilation: float = 0.3
    plane_eps: float = 0.5
    term_eps: float = 1e-4
    alpha_floor: float = 1.0 / 255.0
    alpha_clamp: float = 0.999
    radius_form_cap: float = 0.0
    ste_tau: float = 1e-3
    soft_assignment: bool = False
    soft_tau: float = 1.0
    tile: int = 16

    def effective_near(self, cfg: WaveConfig) -> float:
        return self.near_clip if self.near_clip > 0.0 else 0.2 * cfg.distance


@dataclass
class PropagationOptions:
    pad2x: bool = False
    local_band_limit: bool = False


@dataclass
class PipelineOptions:
    """pipeline.hpp:23-29."""
    raster: RenderSettings = field(default_factory=RenderSettings)
    prop: PropagationOptions = field(default_factory=PropagationOptions)
    lambda_ssim: float = 0.005
    lambda_opacity: float = 1e-4
    use_plain_mse: bool = False


@dataclass
class LossBreakdown:
    """pipeline.hpp:44-48."""
    total: float = 0.0
    recon: float = 0.0
    ssim: float = 0.0
    opacity: float = 0.0
    psnr_mean: float = 0.0
    psnr: List[float] = field(default_factory=list)


@dataclass
class OptimizerConfig:
    """optimizer.hpp:17-31 (Adan; use_adam selects the two-moment fallback)."""
    lr_positions: float = 0.01
    lr_rotations: float = 0.001
    lr_log_scales: float = 0.005
    lr_amplitudes: float = 0.0025
    lr_phases: float = 0.0025
    lr_opacities: float = 0.025
    lr_plane_logits: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.99
    beta3: float = 0.99
    eps: float = 1e-8
    use_adam: bool = False
    schedule_total: int = 20000
    lr_floor: float = 1e-5


def _pad_default():
    return PropagationOptions(pad2x=True)


@dataclass
class PhaseOnlyOptions:
    """phase_only.hpp:22-32 (conversion propagates padded by default)."""
    lambda_ssim: float = 1.0
    prop: PropagationOptions = field(default_factory=_pad_default)
    use_adam: bool = False


@dataclass
class PhaseOnlyHologram:
    """phase_only.hpp:13-19: unit-amplitude hologram e^{j phase}, phase [C, H, W]."""
    phase: np.ndarray

    def field(self, pitch: float = 3.74e-6) -> np.ndarray:
        return np.exp(1j * self.phase) if self.phase.size else self.phase.astype(np.complex128)


@dataclass
class PhaseOnlyResult:
    hologram: PhaseOnlyHologram
    trace: List[float]


@dataclass
class RasterForward:
    layers: List[np.ndarray]          # L x [C, H, W] complex
    t_final: Optional[np.ndarray]     # [L, H, W]
    n_contrib: Optional[np.ndarray]   # [L, H, W]
    projected: Optional[dict]         # field -> [N] arrays (detail::Projected)
    rho: Optional[np.ndarray]         # [N, L]
    touched: Optional[np.ndarray]     # [N]
    entries: Optional[np.ndarray]     # structured: bucket, gidx, depth (detail::Entry)
    bucket_start: Optional[np.ndarray]  # [B + 1] uint32
    tiles_x: int = 0
    tiles_y: int = 0


@dataclass
class PipelineForward:
    raster: Optional[RasterForward]
    hologram: np.ndarray              # [C, H, W] complex
    replayed: Optional[List[np.ndarray]]
    intensities: List[np.ndarray]     # L x [C, H, W]
