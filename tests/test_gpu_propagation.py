"""GPU parity of the propagation operators (fft2/ifft2, transfer_function,
propagate, forward_record, inverse_propagate, intensity) against the oracle and
the reference's own identities (test_propagation.cpp) at the stated precision:
f64 at the reference's tolerances, fp32 within 1e-5 relative."""
import math

import numpy as np
import pytest

from conftest import desk_config, random_bandlimited_field, random_field, rel_l2
from paper_2506_08350_b200._lib import HoloError
from paper_2506_08350_b200.holotypes import PropagationOptions, WaveConfig

pytestmark = pytest.mark.gpu

SIZES = [(48, 48), (64, 48), (13, 17), (30, 42), (256, 256), (1920, 1080), (1080, 1920), (121, 7), (1, 64),
         (64, 1), (1024, 1024)]


@pytest.mark.parametrize("w,h", SIZES)
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_fft2_matches_numpy(gpu_ctx, w, h, precision):
    rng = np.random.default_rng(w * 7 + h)
    x = rng.standard_normal((2, h, w)) + 1j * rng.standard_normal((2, h, w))
    tol = 1e-13 if precision == "f64" else 2e-6
    assert rel_l2(gpu_ctx.fft2(x, False, precision), np.fft.fft2(x)) < tol
    assert rel_l2(gpu_ctx.fft2(x, True, precision), np.fft.ifft2(x)) < tol


def test_fft2_rejects_large_prime(gpu_ctx):
    with pytest.raises(HoloError) as e:
        gpu_ctx.fft2(np.ones((1, 4, 37), complex))
    assert e.value.kind == "config"


@pytest.mark.parametrize("precision,tol", [("f64", 1e-13), ("f32", 2e-5)])
@pytest.mark.parametrize("z", [1.7e-3, -2e-3, 0.0, 4e-3])
def test_propagate_matches_oracle(gpu_ctx, oracle, precision, tol, z):
    cfg = WaveConfig(nx=64, ny=48, num_planes=2)
    u = random_field(cfg, 3)
    assert rel_l2(gpu_ctx.propagate(u, cfg, z, None, precision), oracle.propagate(u, cfg, z)) < tol


@pytest.mark.parametrize("precision,tol", [("f64", 1e-13), ("f32", 2e-5)])
@pytest.mark.parametrize("opt", [PropagationOptions(pad2x=True), PropagationOptions(local_band_limit=True),
                                 PropagationOptions(pad2x=True, local_band_limit=True)])
def test_propagate_options_match_oracle(gpu_ctx, oracle, precision, tol, opt):
    cfg = WaveConfig(nx=48, ny=32, num_planes=2)
    u = random_field(cfg, 5)
    z = 50e-3 if opt.local_band_limit else 1e-3
    assert rel_l2(gpu_ctx.propagate(u, cfg, z, opt, precision), oracle.propagate(u, cfg, z, opt)) < tol


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_transfer_function_matches_oracle(gpu_ctx, oracle, precision):
    cfg = desk_config(64)
    for z in (0.5e-3, 2e-3, -1e-3, 4e-3):
        tol = 1e-13 if precision == "f64" else 2e-5
        assert rel_l2(gpu_ctx.transfer_function(cfg, z, None, precision), oracle.transfer_function(cfg, z)) < tol
    lim = PropagationOptions(local_band_limit=True)
    cfg.wavelengths = (639e-9,)
    a = gpu_ctx.transfer_function(cfg, 50e-3, lim, precision)
    b = oracle.transfer_function(cfg, 50e-3, lim)
    assert np.array_equal(a == 0, b == 0)  # band mask bit-exact


@pytest.mark.parametrize("precision,tol", [("f64", 1e-13), ("f32", 2e-5)])
def test_forward_record_and_inverse_match_oracle(gpu_ctx, oracle, precision, tol):
    for L in (1, 3):
        cfg = WaveConfig(nx=64, ny=64, num_planes=L)
        layers = np.stack([random_field(cfg, 10 + l) for l in range(L)])
        h_gpu = gpu_ctx.forward_record(list(layers), cfg, None, precision)
        h_ref = oracle.forward_record(layers, cfg)
        assert rel_l2(h_gpu, h_ref) < tol
        r_gpu = np.stack(gpu_ctx.inverse_propagate(h_ref, cfg, None, precision))
        assert rel_l2(r_gpu, oracle.inverse_propagate(h_ref, cfg)) < tol
    pad = PropagationOptions(pad2x=True)
    cfg = WaveConfig(nx=32, ny=32, num_planes=2)
    layers = np.stack([random_field(cfg, 20 + l) for l in range(2)])
    assert rel_l2(gpu_ctx.forward_record(list(layers), cfg, pad, precision), oracle.forward_record(layers, cfg, pad)) < tol
    h = oracle.forward_record(layers, cfg, pad)
    assert rel_l2(np.stack(gpu_ctx.inverse_propagate(h, cfg, pad, precision)), oracle.inverse_propagate(h, cfg, pad)) < tol


# ---------------------------------------------------------------- reference identities on the GPU

def test_identities_f64(gpu_ctx):
    # test_propagation.cpp:44-115 at the reference's own tolerances
    cfg = desk_config(128)
    u = random_bandlimited_field(cfg, 11)
    v = gpu_ctx.propagate(gpu_ctx.propagate(u, cfg, 1.7e-3), cfg, -1.7e-3)
    assert np.abs(u - v).max() < 1e-10
    e0 = np.sum(np.abs(u) ** 2)
    for z in (0.4e-3, 2e-3, 4e-3):
        assert abs(np.sum(np.abs(gpu_ctx.propagate(u, cfg, z)) ** 2) - e0) / e0 < 1e-10
    cfg64 = desk_config(64)
    w = random_bandlimited_field(cfg64, 17)
    two = gpu_ctx.propagate(gpu_ctx.propagate(w, cfg64, 0.9e-3), cfg64, 1.4e-3)
    assert np.abs(two - gpu_ctx.propagate(w, cfg64, 2.3e-3)).max() < 1e-10
    assert np.abs(gpu_ctx.propagate(w, cfg64, 0.0) - w).max() < 1e-12
    x, y = random_field(cfg64, 31), random_field(cfg64, 37)
    lhs = np.sum((gpu_ctx.propagate(x, cfg64, 1.9e-3) * np.conj(y)).real)
    rhs = np.sum((x * np.conj(gpu_ctx.propagate(y, cfg64, -1.9e-3))).real)
    assert math.isclose(lhs, rhs, rel_tol=1e-10)
    c1 = desk_config(32)
    c1.wavelengths = (532e-9,)
    z = 1.234e-3
    ph = math.fmod(2 * math.pi * z / 532e-9, 2 * math.pi)
    assert np.allclose(gpu_ctx.propagate(np.ones((1, 32, 32), complex), c1, z), complex(math.cos(ph), math.sin(ph)),
                       rtol=0, atol=1e-9)


def test_identities_f32(gpu_ctx):
    # the same identities at fp32 tolerances (the render path's precision)
    cfg = desk_config(128)
    u = random_bandlimited_field(cfg, 11)
    v = gpu_ctx.propagate(gpu_ctx.propagate(u, cfg, 1.7e-3, None, "f32"), cfg, -1.7e-3, None, "f32")
    assert rel_l2(v, u) < 1e-5
    e0 = np.sum(np.abs(u) ** 2)
    assert abs(np.sum(np.abs(gpu_ctx.propagate(u, cfg, 4e-3, None, "f32")) ** 2) - e0) / e0 < 1e-5
    c1 = desk_config(32)
    c1.wavelengths = (532e-9,)
    z = 1.234e-3
    ph = math.fmod(2 * math.pi * z / 532e-9, 2 * math.pi)
    got = gpu_ctx.propagate(np.ones((1, 32, 32), complex), c1, z, None, "f32")
    assert np.allclose(got, complex(math.cos(ph), math.sin(ph)), rtol=0, atol=2e-6)


def test_forward_record_single_layer_equals_propagate(gpu_ctx):
    # test_propagation.cpp:117-123
    cfg = desk_config(64, 1)
    u = random_field(cfg, 41)
    assert np.abs(gpu_ctx.forward_record([u], cfg) - gpu_ctx.propagate(u, cfg, cfg.distance)).max() < 1e-13


def test_propagate_rejects_channel_mismatch(gpu_ctx):
    with pytest.raises(HoloError) as e:
        gpu_ctx.propagate(np.zeros((1, 32, 32), complex), desk_config(32), 1e-3)
    assert e.value.kind == "config"


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_intensity(gpu_ctx, precision):
    f = np.array([[[3 + 4j, -1 + 2j]]])
    assert np.array_equal(gpu_ctx.intensity(f, precision), np.array([[[25.0, 5.0]]]))
