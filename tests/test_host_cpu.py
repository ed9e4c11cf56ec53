"""Host-side logic on CPU: reference type mirrors and their validation messages,
the synthetic scene generator, HOLOSCENE1 I/O, and the C-ABI library's exports
(no compute calls: there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2506_08350_b200 import _lib
from paper_2506_08350_b200._lib import HoloError
from paper_2506_08350_b200.holotypes import CameraView, GaussianScene, WaveConfig, plane_positions
from paper_2506_08350_b200.scenes import CONFIGS, read_scene, synthetic_scene, write_scene


def test_plane_positions_match_reference_kats():
    # test_field.cpp:13-35
    assert plane_positions(WaveConfig(num_planes=2)) == pytest.approx([0.0, 4e-3], abs=1e-15)
    assert plane_positions(WaveConfig(num_planes=3)) == pytest.approx([0.0, 2e-3, 4e-3], abs=1e-15)
    assert plane_positions(WaveConfig(num_planes=1)) == [2e-3]


def test_plane_positions_equal_oracle(oracle):
    for L in (1, 2, 3, 6, 8, 16):
        cfg = WaveConfig(num_planes=L)
        assert np.array_equal(np.array(plane_positions(cfg)), oracle.plane_positions(cfg))


@pytest.mark.parametrize("kw,msg", [({"pitch": -1.0}, "pixel pitch must be positive"),
                                    ({"wavelengths": (0.0,)}, "wavelengths must be positive"),
                                    ({"num_planes": 0}, "need at least one depth plane"),
                                    ({"nx": 0}, "resolution must be positive"),
                                    ({"num_planes": 4, "volume_depth": 0.0},
                                     "multiple planes need a positive volume depth")])
def test_wave_validation_messages(kw, msg):
    with pytest.raises(HoloError) as e:
        WaveConfig(**kw).validate()
    assert e.value.kind == "config" and str(e.value) == msg


def test_camera_rotation_matches_oracle_order():
    cam = CameraView(pose=(0.1, -0.2, 0.3, 0.01, -0.02, 0.015), width=8, height=8)
    R = cam.rot_cam_to_world()
    assert np.allclose(R @ R.T, np.eye(3), atol=1e-15)
    assert np.array_equal(cam.rot_world_to_cam(), R.T)
    with pytest.raises(HoloError):
        CameraView(width=0, height=4).validate()


def test_scene_validation():
    s = GaussianScene(num_planes=2)
    s.resize(3)
    s.validate()
    s.rotations[1] = 0.0
    with pytest.raises(HoloError, match="degenerate quaternion"):
        s.validate()
    s.resize(3)
    s.amplitudes[2, 1] = -0.1
    with pytest.raises(HoloError, match="non-negative"):
        s.validate()
    s.resize(3)
    s.plane_logits = np.zeros((3, 1))
    with pytest.raises(HoloError, match="inconsistent sizes"):
        s.validate()


def test_synthetic_scene_deterministic_and_in_frustum():
    cfg = CONFIGS["C2"].wave()
    a = synthetic_scene(5000, cfg, 2)
    b = synthetic_scene(5000, cfg, 2)
    for k in ("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases", "plane_logits"):
        assert np.array_equal(getattr(a, k), getattr(b, k))
    a.validate()
    z = a.positions[:, 2]
    assert z.min() >= 0.25 and z.max() < 0.45
    u = a.positions[:, 0] * cfg.nx / z + cfg.nx / 2
    assert u.min() >= 0 and u.max() < cfg.nx
    assert np.allclose(np.linalg.norm(a.rotations, axis=1), 1.0)
    assert np.bincount(a.plane_logits.argmax(1)).tolist() == [834, 834, 833, 833, 833, 833]


def test_holoscene_round_trip(tmp_path):
    cfg = WaveConfig(nx=32, ny=32, num_planes=3)
    s = synthetic_scene(50, cfg, 4)
    p = tmp_path / "s.holoscene"
    write_scene(str(p), s)
    r = read_scene(str(p))
    for k in ("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases", "plane_logits"):
        assert np.array_equal(getattr(r, k), getattr(s, k))
    raw = p.read_bytes()
    assert raw[:10] == b"HOLOSCENE1"
    bad = tmp_path / "bad"
    bad.write_bytes(b"definitely not a scene")
    with pytest.raises(HoloError) as e:
        read_scene(str(bad))
    assert e.value.kind == "io"
    trunc = tmp_path / "trunc"
    trunc.write_bytes(raw[:-8])
    with pytest.raises(HoloError, match="truncated"):
        read_scene(str(trunc))


def _declared(header):
    text = open(header).read()
    return sorted(set(re.findall(r"\b(holo_[a-z0-9_]+)\s*\(", text)))


def test_c_abi_exports_every_declared_symbol():
    decl = _declared(os.path.join(ROOT, "include", "holo_cuda.h"))
    assert len(decl) >= 25
    assert os.path.exists(_lib.LIB_PATH), "libholo_cuda.so must be built (__graft_entry__.build())"
    lib = ctypes.CDLL(_lib.LIB_PATH)  # loads without a GPU (cudart resolves lazily)
    missing = [n for n in decl if not hasattr(lib, n)]
    assert not missing, missing
    L = _lib.lib()
    assert L.holo_abi_version() == 1
    assert L.holo_fft_supported(1920) == 1 and L.holo_fft_supported(1080) == 1
    assert L.holo_fft_supported(37) == 0


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2506_08350_b200 import api

    with pytest.raises(HoloError):
        api.Context(0)
