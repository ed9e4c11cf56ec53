"""Deterministic synthetic scenes and the BASELINE configurations.

The reference's own bench scene (holo_main.cpp:53-81, ``demo_scene``) packs
every splat into ~20 central tiles at 1080p, so the benchmark scenes follow the
generator SURVEY.md 8(d) specifies instead: a counter-based RNG (splitmix64,
u = (x >> 11) 2^-53, Box-Muller normals) so the oracle and the GPU consume
identical f64 bytes; positions fill the view frustum at z ~ U(0.25, 0.45) m for
a camera at the origin with focal = W px; quaternions are normalised N(0,1)^4
(helpers.hpp:91-93); log scales give a projected sigma log-uniform in
[0.5, 3] px; amplitudes U(0.2, 1); opacity logits U(-2, 2); phases U(0, 2 pi);
plane logits 0.1 l with 2.0 at l = i mod L (holo_main.cpp:77-78).

HOLOSCENE1 I/O follows scene_io.cpp:29-95 (10-byte magic, u32 header length,
JSON header, then the seven f64 arrays in declaration order).
"""
from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

from .holotypes import CameraView, GaussianScene, WaveConfig

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _uniform(seed: int, idx: np.ndarray, k: int) -> np.ndarray:
    """u in [0, 1) for draw k of Gaussian idx: splitmix64(key + 32 idx + k) >> 11 * 2^-53."""
    key = splitmix64(np.array([seed], dtype=np.uint64))[0]
    with np.errstate(over="ignore"):
        ctr = key + idx.astype(np.uint64) * np.uint64(32) + np.uint64(k)
    return (splitmix64(ctr) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _normal_pair(seed: int, idx: np.ndarray, k: int) -> Tuple[np.ndarray, np.ndarray]:
    u1 = 1.0 - _uniform(seed, idx, k)  # (0, 1]
    u2 = _uniform(seed, idx, k + 1)
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(2.0 * math.pi * u2), r * np.sin(2.0 * math.pi * u2)


def synthetic_scene(n: int, cfg: WaveConfig, seed: int, focal_px: float = None) -> GaussianScene:
    W, H, L = cfg.nx, cfg.ny, cfg.num_planes
    f = float(W if focal_px is None else focal_px)
    i = np.arange(n, dtype=np.int64)
    z = 0.25 + 0.2 * _uniform(seed, i, 0)
    x = (_uniform(seed, i, 1) - 0.5) * W * z / f
    y = (_uniform(seed, i, 2) - 0.5) * H * z / f
    q0, q1 = _normal_pair(seed, i, 3)
    q2, q3 = _normal_pair(seed, i, 5)
    q = np.stack([q0, q1, q2, q3], axis=1)
    norm = np.sqrt(((q[:, 0] * q[:, 0] + q[:, 1] * q[:, 1]) + q[:, 2] * q[:, 2]) + q[:, 3] * q[:, 3])
    ok = norm > 1e-9
    q = np.where(ok[:, None], q / np.where(ok, norm, 1.0)[:, None], np.array([1.0, 0.0, 0.0, 0.0]))
    sig_px = np.stack([np.exp(math.log(0.5) + (math.log(3.0) - math.log(0.5)) * _uniform(seed, i, 7 + d))
                       for d in range(3)], axis=1)
    log_scales = np.log(sig_px * 0.35 / f)
    amps = np.stack([0.2 + 0.8 * _uniform(seed, i, 10 + d) for d in range(3)], axis=1)
    opac = -2.0 + 4.0 * _uniform(seed, i, 13)
    phases = np.stack([2.0 * math.pi * _uniform(seed, i, 14 + d) for d in range(3)], axis=1)
    logits = np.tile(0.1 * np.arange(L, dtype=np.float64), (n, 1))
    logits[i, i % L] = 2.0
    s = GaussianScene(num_planes=L)
    s.positions = np.ascontiguousarray(np.stack([x, y, z], axis=1))
    s.rotations = np.ascontiguousarray(q)
    s.log_scales = np.ascontiguousarray(log_scales)
    s.amplitudes = np.ascontiguousarray(amps)
    s.opacity_logits = np.ascontiguousarray(opac)
    s.phases = np.ascontiguousarray(phases)
    s.plane_logits = np.ascontiguousarray(logits)
    return s


def front_camera(cfg: WaveConfig, focal: float = None, yaw: float = 0.0) -> CameraView:
    return CameraView(pose=(0.0, 0.0, 0.0, 0.0, float(yaw), 0.0), focal_px=float(cfg.nx if focal is None else focal),
                      width=cfg.nx, height=cfg.ny)


@dataclass
class BenchConfig:
    name: str
    n: int
    nx: int
    ny: int
    planes: int
    wavelengths: Tuple[float, ...]
    seed: int
    views: int = 1
    shard: str = "planes"  # multi-GPU split: "planes", "views" or "planes_views" (bench.py)

    def wave(self) -> WaveConfig:
        return WaveConfig(nx=self.nx, ny=self.ny, pitch=3.74e-6, wavelengths=tuple(self.wavelengths),
                          distance=2e-3, volume_depth=4e-3, num_planes=self.planes)

    def cameras(self) -> List[CameraView]:
        cfg = self.wave()
        if self.views == 1:
            return [front_camera(cfg)]
        return [front_camera(cfg, yaw=-0.1 + 0.2 * k / (self.views - 1)) for k in range(self.views)]


RGB = (638e-9, 520e-9, 450e-9)
CONFIGS = {
    "C1": BenchConfig("C1", 10_000, 256, 256, 3, (515e-9,), 1),
    "C2": BenchConfig("C2", 100_000, 1024, 1024, 6, RGB, 2),
    "C3": BenchConfig("C3", 1_000_000, 1920, 1080, 8, RGB, 3),
    "C4": BenchConfig("C4", 1_000_000, 1024, 1024, 6, RGB, 4, views=64, shard="views"),
    # BASELINE names planes x views for C5 without a view count: a batch of 8 views
    # (yaw -0.1 .. +0.1 rad), 2 plane ranks x 4 view groups on 8 GPUs
    "C5": BenchConfig("C5", 3_000_000, 3840, 2160, 16, RGB, 5, views=8, shard="planes_views"),
}


# ---------------------------------------------------------------- HOLOSCENE1

_MAGIC = b"HOLOSCENE1"


def write_scene(path: str, s: GaussianScene) -> None:
    """scene_io.cpp:29-58."""
    s.validate()
    header = {"L": int(s.num_planes), "N": int(s.size()),
              "units": {"amplitudes": "linear", "opacities": "logit", "phases": "rad", "plane_logits": "logit",
                        "positions": "m", "rotations": "unit_quaternion_wxyz", "scales": "log_m"}}
    hs = json.dumps(header, separators=(",", ":"), sort_keys=True).encode()
    with open(path, "wb") as fp:
        fp.write(_MAGIC)
        fp.write(struct.pack("<I", len(hs)))
        fp.write(hs)
        for a in (s.positions, s.rotations, s.log_scales, s.amplitudes, s.opacity_logits, s.phases, s.plane_logits):
            fp.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def read_scene(path: str) -> GaussianScene:
    """scene_io.cpp:60-95."""
    from ._lib import HoloError

    with open(path, "rb") as fp:
        if fp.read(10) != _MAGIC:
            raise HoloError("io", f"bad magic, not a HOLOSCENE1 file: {path}")
        (hlen,) = struct.unpack("<I", fp.read(4))
        if hlen == 0 or hlen > (1 << 20):
            raise HoloError("io", f"implausible header length in {path}")
        header = json.loads(fp.read(hlen))
        n, L = int(header["N"]), int(header["L"])
        if L < 1 or n > (1 << 26):
            raise HoloError("io", f"implausible scene dimensions in {path}")

        def arr(count, shape):
            b = fp.read(8 * count)
            if len(b) != 8 * count:
                raise HoloError("io", f"truncated payload: {path}")
            return np.frombuffer(b, dtype="<f8").reshape(shape).copy()

        s = GaussianScene(num_planes=L)
        s.positions = arr(3 * n, (n, 3))
        s.rotations = arr(4 * n, (n, 4))
        s.log_scales = arr(3 * n, (n, 3))
        s.amplitudes = arr(3 * n, (n, 3))
        s.opacity_logits = arr(n, (n,))
        s.phases = arr(3 * n, (n, 3))
        s.plane_logits = arr(n * L, (n, L))
    s.validate()
    return s
