"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and run on a B200 box; the
rest runs on CPU (the oracle, host logic, C-ABI symbol checks, gloo sharding)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_2506_08350_b200.holotypes import (CameraView, GaussianScene, RenderSettings,  # noqa: E402
                                             WaveConfig)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs libholo_cuda kernels")
    config.addinivalue_line("markers", "slow: full-size parity (seconds of oracle time)")


@pytest.fixture(scope="session")
def oracle():
    """The plain-C restatement (always built by __graft_entry__.build())."""
    return Oracle("restate")


@pytest.fixture(scope="session")
def ref_oracle():
    """The reference itself, compiled from /root/reference (oracle/_ref)."""
    if not Oracle.available("ref"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2506_08350_b200.api import Context

    return Context(0)


# ------------------------------------------------------------ reference test helpers (tests/helpers.hpp)

def desk_config(n=128, planes=2):
    """helpers.hpp:14-24."""
    return WaveConfig(nx=n, ny=n, pitch=3.74e-6, wavelengths=(639e-9, 532e-9, 473e-9), distance=2e-3,
                      volume_depth=4e-3, num_planes=planes)


def front_camera(cfg, focal=150.0):
    """helpers.hpp:64-70."""
    return CameraView(focal_px=focal, width=cfg.nx, height=cfg.ny)


def mild_posed_camera(cfg):
    """helpers.hpp:115-119."""
    cam = front_camera(cfg)
    cam.pose = (0.005, -0.003, -0.02, 0.01, -0.02, 0.015)
    return cam


def random_field(cfg, seed, rng=None):
    rng = np.random.default_rng(seed)
    c, h, w = cfg.channels(), cfg.ny, cfg.nx
    return rng.standard_normal((c, h, w)) + 1j * rng.standard_normal((c, h, w))


def random_bandlimited_field(cfg, seed):
    """helpers.hpp:36-55 (numpy FFT; every bin outside 1/lambda^2 zeroed)."""
    f = random_field(cfg, seed)
    for ch, lam in enumerate(cfg.wavelengths):
        F = np.fft.fft2(f[ch])
        ky = np.fft.fftfreq(cfg.ny) * cfg.ny
        kx = np.fft.fftfreq(cfg.nx) * cfg.nx
        fy = ky / (cfg.ny * cfg.pitch)
        fx = kx / (cfg.nx * cfg.pitch)
        mask = fx[None, :] ** 2 + fy[:, None] ** 2 > 1.0 / lam ** 2
        F[mask] = 0
        f[ch] = np.fft.ifft2(F)
    return f


def random_scene(n, cfg, seed):
    """helpers.hpp:74-101 in spirit (numpy RNG, same distributions)."""
    rng = np.random.default_rng(seed)
    s = GaussianScene(num_planes=cfg.num_planes)
    s.positions = np.stack([rng.uniform(-0.05, 0.05, n), rng.uniform(-0.05, 0.05, n), rng.uniform(0.25, 0.45, n)], 1)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    s.rotations = q
    s.log_scales = np.log(rng.uniform(0.003, 0.012, (n, 3)))
    s.amplitudes = rng.uniform(0.2, 1.0, (n, 3))
    s.opacity_logits = rng.uniform(-2.0, 2.0, n)
    s.phases = rng.uniform(0.0, 2 * np.pi, (n, 3))
    s.plane_logits = rng.standard_normal((n, cfg.num_planes))
    return s


def overlapping_scene(n, cfg, seed):
    """helpers.hpp:123-132."""
    s = random_scene(n, cfg, seed)
    s.positions[:, :2] *= 0.25
    L = cfg.num_planes
    s.plane_logits = np.tile(0.1 * np.arange(L, dtype=np.float64), (n, 1))
    s.plane_logits[np.arange(n), np.arange(n) % L] = 2.0
    return s


def single_scene(n, planes):
    s = GaussianScene(num_planes=planes)
    s.resize(n)
    return s


def rel_l2(a, b):
    a, b = np.asarray(a), np.asarray(b)
    d = float(np.linalg.norm(b.ravel()))
    return float(np.linalg.norm((a - b).ravel())) / (d if d > 0 else 1.0)
