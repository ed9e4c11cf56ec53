"""The reference's own known-answer tests and identities, run against the CPU
oracles (CPU only).  Each test names the reference test it ports
(/root/reference/proj/tests/*.cpp); both the C restatement and -- where built --
the reference compiled from its sources must pass them.  This pins the oracle
before it is trusted as the GPU parity checker."""
import math

import numpy as np
import pytest

from conftest import (desk_config, front_camera, overlapping_scene, random_bandlimited_field, random_field,
                      random_scene, single_scene)
from oracle.oracle import Oracle, OracleError
from paper_2506_08350_b200.holotypes import PropagationOptions, RenderSettings, WaveConfig

BACKENDS = ["restate", "ref"]


@pytest.fixture(params=BACKENDS)
def ora(request):
    if not Oracle.available(request.param):
        pytest.skip(f"oracle backend {request.param} not built")
    return Oracle(request.param)


# ------------------------------------------------------------------ test_field.cpp

def test_plane_positions_kats(oracle):
    # test_field.cpp:13-45
    assert np.allclose(oracle.plane_positions(desk_config(64, 2)), [0.0, 4e-3], atol=1e-15)
    assert np.allclose(oracle.plane_positions(desk_config(64, 3)), [0.0, 2e-3, 4e-3], atol=1e-15)
    assert list(oracle.plane_positions(desk_config(64, 1))) == [2e-3]
    cfg = desk_config(32, 5)
    cfg.distance, cfg.volume_depth = 3.1e-3, 1.7e-3
    z = oracle.plane_positions(cfg)
    assert np.allclose(np.diff(z), 1.7e-3 / 4, rtol=1e-12)
    assert math.isclose(0.5 * (z[0] + z[-1]), 3.1e-3, rel_tol=1e-12)


@pytest.mark.parametrize("field,value", [("pitch", -1.0), ("wavelengths", (0.0,)), ("num_planes", 0), ("nx", 0)])
def test_config_validation_rejects(oracle, field, value):
    # test_field.cpp:47-64
    cfg = desk_config()
    setattr(cfg, field, value)
    with pytest.raises(OracleError) as e:
        oracle.plane_positions(cfg)
    assert e.value.kind == "config"
    cfg = desk_config()
    cfg.num_planes, cfg.volume_depth = 4, 0.0
    with pytest.raises(OracleError):
        oracle.plane_positions(cfg)


# ------------------------------------------------------------------ test_propagation.cpp

def test_tf_unit_modulus_in_band(ora):
    # test_propagation.cpp:10-32
    cfg = desk_config(64)
    for z in (0.5e-3, 2e-3, -1e-3):
        tf = ora.transfer_function(cfg, z)
        assert np.allclose(np.abs(tf), 1.0, rtol=0, atol=1e-12)  # every bin is in band at this pitch


def test_tf_conjugate_symmetry(ora):
    # test_propagation.cpp:34-42
    cfg = desk_config(32)
    a = ora.transfer_function(cfg, 1.3e-3)
    b = ora.transfer_function(cfg, -1.3e-3)
    assert np.allclose(a, np.conj(b), rtol=1e-15, atol=1e-15)


def test_round_trip(ora):
    # test_propagation.cpp:44-49
    cfg = desk_config(128)
    u = random_bandlimited_field(cfg, 11)
    v = ora.propagate(ora.propagate(u, cfg, 1.7e-3), cfg, -1.7e-3)
    assert np.abs(u - v).max() < 1e-10


def test_energy_conservation(ora):
    # test_propagation.cpp:51-59
    cfg = desk_config(128)
    u = random_bandlimited_field(cfg, 13)
    e0 = np.sum(np.abs(u) ** 2)
    for z in (0.4e-3, 2e-3, 4e-3):
        assert abs(np.sum(np.abs(ora.propagate(u, cfg, z)) ** 2) - e0) / e0 < 1e-10


def test_composition(ora):
    # test_propagation.cpp:61-67
    cfg = desk_config(64)
    u = random_bandlimited_field(cfg, 17)
    two = ora.propagate(ora.propagate(u, cfg, 0.9e-3), cfg, 1.4e-3)
    one = ora.propagate(u, cfg, 2.3e-3)
    assert np.abs(two - one).max() < 1e-10


def test_zero_distance_identity(ora):
    # test_propagation.cpp:69-74
    cfg = desk_config(64)
    u = random_bandlimited_field(cfg, 19)
    assert np.abs(ora.propagate(u, cfg, 0.0) - u).max() < 1e-12


def test_linearity(ora):
    # test_propagation.cpp:76-89
    cfg = desk_config(32)
    a, b = random_field(cfg, 23), random_field(cfg, 29)
    s = 0.7 - 1.2j
    lhs = ora.propagate(s * a + b, cfg, 1.1e-3)
    rhs = s * ora.propagate(a, cfg, 1.1e-3) + ora.propagate(b, cfg, 1.1e-3)
    assert np.abs(lhs - rhs).max() < 1e-10


def test_adjoint(ora):
    # test_propagation.cpp:93-101
    cfg = desk_config(64)
    x, y = random_field(cfg, 31), random_field(cfg, 37)
    lhs = np.sum((ora.propagate(x, cfg, 1.9e-3) * np.conj(y)).real)
    rhs = np.sum((x * np.conj(ora.propagate(y, cfg, -1.9e-3))).real)
    assert math.isclose(lhs, rhs, rel_tol=1e-10)


def test_constant_field_on_axis_phase(ora):
    # test_propagation.cpp:103-115
    cfg = desk_config(32)
    cfg.wavelengths = (532e-9,)
    u = np.ones((1, 32, 32), dtype=complex)
    z = 1.234e-3
    v = ora.propagate(u, cfg, z)
    ph = math.fmod(2 * math.pi * z / 532e-9, 2 * math.pi)
    assert np.allclose(v, complex(math.cos(ph), math.sin(ph)), rtol=0, atol=1e-9)


def test_forward_record_one_layer_equals_propagate(ora):
    # test_propagation.cpp:117-123 (exact equality)
    cfg = desk_config(64, 1)
    u = random_field(cfg, 41)
    assert np.array_equal(ora.forward_record(u[None], cfg), ora.propagate(u, cfg, cfg.distance))


def test_record_then_inverse_recovers(ora):
    # test_propagation.cpp:125-134
    cfg = desk_config(64, 1)
    u = random_bandlimited_field(cfg, 43)
    stack = ora.inverse_propagate(ora.forward_record(u[None], cfg), cfg)
    assert stack.shape[0] == 1 and np.abs(stack[0] - u).max() < 1e-10


def test_inverse_returns_one_field_per_plane(ora):
    # test_propagation.cpp:136-145
    cfg = desk_config(32, 3)
    assert ora.inverse_propagate(random_field(cfg, 47), cfg).shape == (3, 3, 32, 32)


def test_padded_close_for_compact_fields(ora):
    # test_propagation.cpp:147-162
    cfg = desk_config(128)
    cfg.wavelengths = (532e-9,)
    y, x = np.mgrid[0:128, 0:128]
    u = np.exp(-((x - 64.0) ** 2 + (y - 64.0) ** 2) / (2 * 64.0))[None].astype(complex)
    a = ora.propagate(u, cfg, 0.5e-3)
    b = ora.propagate(u, cfg, 0.5e-3, PropagationOptions(pad2x=True))
    assert np.abs(a - b).max() < 1e-6


def test_local_band_limit(ora):
    # test_propagation.cpp:164-183
    cfg = desk_config(64)
    cfg.wavelengths = (639e-9,)
    plain = ora.transfer_function(cfg, 50e-3)
    lim = ora.transfer_function(cfg, 50e-3, PropagationOptions(local_band_limit=True))
    zeroed = (np.abs(lim) == 0) & (np.abs(plain) > 0)
    assert zeroed.sum() > 0 and (~zeroed).sum() > 0
    assert np.array_equal(lim[~zeroed], plain[~zeroed])


def test_propagate_rejects_channel_mismatch(ora):
    # propagation.cpp:94-95
    cfg = desk_config(32)
    with pytest.raises(OracleError) as e:
        ora.propagate(np.zeros((1, 32, 32), complex), cfg, 1e-3)
    assert e.value.kind == "config"


# ------------------------------------------------------------------ test_scene.cpp

def test_covariance_kats(oracle):
    # test_scene.cpp:15-52
    s = oracle.covariance_3d([1, 0, 0, 0], np.log([0.5, 0.25, 2.0]))
    assert np.allclose(np.diag(s), [0.25, 0.0625, 4.0], rtol=1e-14)
    assert np.abs(s - np.diag(np.diag(s))).max() < 1e-15
    c, sn = math.cos(math.pi / 4), math.sin(math.pi / 4)
    s = oracle.covariance_3d([c, 0, 0, sn], np.log([3.0, 1.0, 0.5]))
    assert np.allclose(np.diag(s), [1.0, 9.0, 0.25], rtol=1e-12)
    rng = np.random.default_rng(7)
    for _ in range(10):
        q = rng.standard_normal(4)
        ls = 0.2 * rng.standard_normal(3)
        a, b = oracle.covariance_3d(q, ls), oracle.covariance_3d(-3.0 * q, ls)
        assert np.abs(a - b).max() < 1e-12
        assert np.abs(a - a.T).max() < 1e-14 and np.linalg.det(a) > 0


def test_argmax_ties_lowest(oracle):
    # test_scene.cpp:54-64
    assert oracle.ste_argmax([0.7, 0.7, 0.7, 0.2]) == 0
    assert oracle.ste_argmax([-1.0, 0.5, 2.0]) == 2


# ------------------------------------------------------------------ test_rasterizer.cpp

def one_gaussian(z=0.3, off=None, logit=0.5, planes=1):
    s = single_scene(1, planes)
    return s


def test_one_gaussian_lands_where_pinhole_says(ora):
    # test_rasterizer.cpp:76-115
    cfg = desk_config(32, 1)
    cam = front_camera(cfg)
    s = single_scene(1, 1)
    s.positions = np.array([[0.01, -0.005, 0.3]])
    q = np.array([0.9, 0.1, -0.3, 0.2])
    s.rotations = (q / np.linalg.norm(q))[None]
    s.log_scales = np.log([[0.004, 0.006, 0.003]])
    s.amplitudes = np.array([[0.8, 0.5, 0.3]])
    s.phases = np.array([[0.3, 1.2, 2.5]])
    s.opacity_logits = np.array([0.5])
    r = ora.raster_forward(s, cam, cfg)
    assert math.isclose(r.projected["mu_x"][0], 21.0, rel_tol=1e-12)
    assert math.isclose(r.projected["mu_y"][0], 13.5, rel_tol=1e-12)
    assert r.touched[0] == 1 and r.layers[0, 0, 0, 0] == 0
    assert r.n_contrib[0, 13, 21] == 1


def centred_scene(n, logits, phases=None, amps=None):
    cfg = desk_config(32, 1)
    cam = front_camera(cfg)
    z = 0.3
    off = 0.5 * z / cam.focal_px
    s = single_scene(n, 1)
    s.positions = np.tile([off, off, z], (n, 1))
    s.log_scales = np.full((n, 3), np.log(0.004))
    s.amplitudes = np.ones((n, 3)) if amps is None else amps
    s.opacity_logits = np.array(logits, dtype=float)
    if phases is not None:
        s.phases = np.array(phases, dtype=float)
    return cfg, cam, s


def test_blending_hand_computed(ora):
    # test_rasterizer.cpp:117-157
    cfg, cam, s = centred_scene(1, [math.log(0.8 / 0.2)])
    r = ora.raster_forward(s, cam, cfg)
    assert abs(r.layers[0, 0, 16, 16] - 0.8) < 1e-12
    assert math.isclose(r.t_final[0, 16, 16], 0.2, rel_tol=1e-12)
    cfg, cam, s = centred_scene(1, [math.log(0.8 / 0.2)], phases=[[math.pi / 2] * 3])
    assert abs(ora.raster_forward(s, cam, cfg).layers[0, 0, 16, 16] - 0.8j) < 1e-12
    cfg, cam, s = centred_scene(2, [0.0, 0.0], phases=[[0, 0, 0], [math.pi] * 3])
    r = ora.raster_forward(s, cam, cfg)
    assert abs(r.layers[0, 0, 16, 16] - 0.25) < 1e-12
    assert math.isclose(r.t_final[0, 16, 16], 0.25, rel_tol=1e-12)


def test_plane_routing(ora):
    # test_rasterizer.cpp:159-188
    cfg = desk_config(32, 2)
    cam = front_camera(cfg)
    s = single_scene(2, 2)
    s.positions = np.array([[-0.02, 0.0, 0.3], [0.02, 0.0, 0.3]])
    s.log_scales = np.full((2, 3), np.log(0.004))
    s.amplitudes = np.full((2, 3), 0.7)
    s.opacity_logits = np.array([1.0, 1.0])
    s.plane_logits = np.array([[2.0, 0.0], [0.0, 2.0]])
    r = ora.raster_forward(s, cam, cfg)
    assert list(r.projected["plane"]) == [0, 1]
    assert abs(r.layers[0, 0, 16, 6]) > 0.1 and abs(r.layers[1, 0, 16, 6]) == 0
    assert abs(r.layers[1, 0, 16, 26]) > 0.1 and abs(r.layers[0, 0, 16, 26]) == 0
    assert np.array_equal(r.rho.sum(1), [1.0, 1.0])


def test_equal_depth_tie_by_index(ora):
    # test_rasterizer.cpp:222-242
    cfg = desk_config(32, 1)
    cam = front_camera(cfg)
    s = single_scene(2, 1)
    s.positions = np.array([[0.0, 0.0, 0.3], [0.0, 0.0, 0.3]])
    s.log_scales = np.full((2, 3), np.log(0.005))
    s.amplitudes = np.ones((2, 3))
    s.phases = np.array([[0.0] * 3, [math.pi / 2] * 3])
    r = ora.raster_forward(s, cam, cfg)
    b = int(r.bucket_start[np.searchsorted(r.bucket_start, 0, side="right") - 1])
    first = r.entry_gidx[r.entry_bucket == r.entry_bucket[0]]
    assert list(first) == [0, 1]


def test_tiled_equals_brute_force_bitwise(ora):
    # test_rasterizer.cpp:244-255
    cfg = desk_config(48, 2)
    cam = front_camera(cfg)
    st = RenderSettings(term_eps=0.0)
    for seed in range(1, 7):
        s = random_scene(30, cfg, seed)
        assert np.array_equal(ora.raster_forward(s, cam, cfg, st).layers, ora.brute_force_forward(s, cam, cfg, st))


def test_early_termination_bound(ora):
    # test_rasterizer.cpp:257-275
    cfg = desk_config(48, 2)
    cam = front_camera(cfg)
    fired = False
    for seed in (11, 12, 13):
        # the reference draws 60 splats with mt19937; 200 numpy-drawn ones make sure
        # enough of them stack up for the transmittance floor to trigger
        s = random_scene(200, cfg, seed)
        s.opacity_logits = np.full(200, 3.0)
        got = ora.raster_forward(s, cam, cfg).layers
        exact = ora.brute_force_forward(s, cam, cfg, RenderSettings(term_eps=0.0))
        assert np.abs(got - exact).max() <= 1e-4 * np.abs(exact).max() + 1e-15
        fired |= not np.array_equal(got, ora.raster_forward(s, cam, cfg, RenderSettings(term_eps=0.0)).layers)
    assert fired


def test_near_plane_culling(ora):
    # test_rasterizer.cpp:307-325
    cfg = desk_config(32, 1)
    cam = front_camera(cfg)
    s = single_scene(2, 1)
    s.positions = np.array([[0.0, 0.0, 1e-4], [0.0, 0.0, -0.5]])
    s.log_scales = np.full((2, 3), np.log(0.005))
    s.amplitudes = np.ones((2, 3))
    s.opacity_logits = np.array([2.0, 2.0])
    r = ora.raster_forward(s, cam, cfg)
    assert list(r.projected["valid"]) == [0, 0] and list(r.touched) == [0, 0]
    assert not np.any(r.layers)


def test_opacity_clamp(ora):
    # test_rasterizer.cpp:327-344
    cfg = desk_config(32, 1)
    cam = front_camera(cfg)
    s = single_scene(1, 1)
    s.positions = np.array([[0.0, 0.0, 0.3]])
    s.log_scales = np.full((1, 3), np.log(0.05))
    s.amplitudes = np.ones((1, 3))
    s.opacity_logits = np.array([40.0])
    r = ora.raster_forward(s, cam, cfg)
    assert r.t_final[0, 16, 16] >= 1.0 - 0.999
    assert np.abs(r.layers).max() <= 0.999 + 1e-12


def test_rejects_mismatched_shapes(ora):
    # test_rasterizer.cpp:346-358
    cfg = desk_config(32, 2)
    cam = front_camera(cfg)
    s = random_scene(3, cfg, 1)
    s.num_planes = 1
    s.plane_logits = s.plane_logits[:, :1]
    with pytest.raises(OracleError):
        ora.raster_forward(s, cam, cfg)
    s2 = random_scene(3, cfg, 1)
    bad = front_camera(cfg)
    bad.width = 16
    with pytest.raises(OracleError):
        ora.raster_forward(s2, bad, cfg)


# ------------------------------------------------------------------ test_pipeline.cpp

def test_pipeline_shapes_and_intensity(ora):
    # test_pipeline.cpp:35-55
    cfg = WaveConfig(nx=32, ny=32, num_planes=2)
    r = ora.pipeline_forward(random_scene(6, cfg, 1), front_camera(cfg), cfg)
    assert r.hologram.shape == (3, 32, 32) and r.replayed.shape == (2, 3, 32, 32)
    assert np.array_equal(r.intensities, np.abs(r.replayed) ** 2) or np.allclose(
        r.intensities, r.replayed.real ** 2 + r.replayed.imag ** 2, rtol=0, atol=0)


def test_amplitude_doubling_quadruples_intensity(ora):
    # test_pipeline.cpp:171-187
    cfg = WaveConfig(nx=32, ny=32, num_planes=2)
    cam = front_camera(cfg)
    s = overlapping_scene(8, cfg, 5)
    a = ora.pipeline_forward(s, cam, cfg)
    s.amplitudes = 2.0 * s.amplitudes
    b = ora.pipeline_forward(s, cam, cfg)
    assert np.allclose(b.intensities, 4.0 * a.intensities, rtol=1e-10, atol=1e-14)


def test_restatement_equals_reference_bitwise(ref_oracle, oracle):
    """The restatement reproduces the reference bit for bit (all outputs)."""
    from paper_2506_08350_b200.scenes import front_camera as fc, synthetic_scene

    for (n, W, H, L, wl, seed, st) in [(300, 64, 48, 3, (639e-9, 532e-9, 473e-9), 1, RenderSettings()),
                                       (2000, 128, 96, 2, (639e-9, 532e-9, 473e-9), 2, RenderSettings(tile=8)),
                                       (500, 64, 64, 3, (515e-9,), 3, RenderSettings()),
                                       (200, 48, 48, 3, (639e-9, 532e-9, 473e-9), 4,
                                        RenderSettings(soft_assignment=True, term_eps=0.0, alpha_floor=0.0))]:
        cfg = WaveConfig(nx=W, ny=H, wavelengths=wl, num_planes=L)
        sc = synthetic_scene(n, cfg, seed)
        cam = fc(cfg)
        a = ref_oracle.pipeline_forward(sc, cam, cfg, st)
        b = oracle.pipeline_forward(sc, cam, cfg, st)
        for k in ("hologram", "replayed", "intensities"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), k
        for k in ("layers", "t_final", "n_contrib", "entry_gidx", "entry_bucket", "entry_depth", "bucket_start",
                  "rho", "touched"):
            assert np.array_equal(getattr(a.raster, k), getattr(b.raster, k)), k
        for k, v in a.raster.projected.items():
            assert np.array_equal(v, b.raster.projected[k]), k
