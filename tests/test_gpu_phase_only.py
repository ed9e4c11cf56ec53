"""GPU phase-only conversion (phase_only.cpp) against the reference build and the
reference's own test cases (tests/test_phase_only.cpp).

Bars: the GPU path is f64 like the reference (FFT sweeps with the transfer
function fused, tree-ordered matching sums), so phase_only_loss and its gradient
agree with the reference to 1e-10 relative, and a conversion's trace follows the
reference's trace (same backtracking decisions) to 1e-8 relative over tens of
iterations."""
import numpy as np
import pytest

from conftest import front_camera, overlapping_scene, rel_l2
from oracle.oracle import Oracle
from paper_2506_08350_b200 import api
from paper_2506_08350_b200._lib import HoloError
from paper_2506_08350_b200.holotypes import PhaseOnlyOptions, PipelineOptions, PropagationOptions, WaveConfig

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not Oracle.available("ref"):
        pytest.skip("reference build (oracle/_ref) not available")
    return Oracle("ref")


def grid(n, planes, wavelengths=(639e-9, 532e-9, 473e-9)):
    return WaveConfig(nx=n, ny=n, wavelengths=wavelengths, num_planes=planes)


def scene_hologram(ctx, cfg, seed, gaussians):
    """test_phase_only.cpp:23-26."""
    return api.pipeline_forward(overlapping_scene(gaussians, cfg, seed), front_camera(cfg), cfg, PipelineOptions(),
                                ctx=ctx, raster=False, replayed=False).hologram


def perturbed_arg(P, seed):
    rng = np.random.default_rng(seed)
    return np.angle(P) + rng.uniform(-0.3, 0.3, P.shape)


# ------------------------------------------------------------------ reference tests

def test_unit_amplitude_fixed_point(gpu_ctx):
    """test_phase_only.cpp:44-63."""
    cfg = grid(32, 2)
    rng = np.random.default_rng(11)
    P = np.exp(1j * rng.uniform(0.0, 2 * np.pi, (3, 32, 32)))
    ext = api.convert_phase_only(P, cfg, 0, ctx=gpu_ctx)
    assert len(ext.trace) == 1 and ext.trace[0] < 1e-20
    assert np.array_equal(ext.hologram.phase, np.angle(P))  # pure extraction, bit for bit
    opt = api.convert_phase_only(P, cfg, 4, ctx=gpu_ctx)
    assert len(opt.trace) == 5
    assert api.phase_only_loss(P, opt.hologram.phase, cfg, ctx=gpu_ctx) < 1e-20


def test_conversion_reduces_loss(gpu_ctx):
    """test_phase_only.cpp:65-89."""
    cfg = grid(32, 1)
    P = scene_hologram(gpu_ctx, cfg, 33, 8)
    res = api.convert_phase_only(P, cfg, 120, ctx=gpu_ctx)
    assert len(res.trace) == 121
    init, best = res.trace[0], min(res.trace)
    assert init > 0.1 and best < 0.15 * init
    assert api.phase_only_loss(P, res.hologram.phase, cfg, ctx=gpu_ctx) == best
    f = res.hologram.field(cfg.pitch)
    assert np.max(np.abs(np.abs(f) - 1.0)) <= 4.0 * np.finfo(float).eps


def test_trace_starts_at_extraction_loss(gpu_ctx):
    """test_phase_only.cpp:91-101."""
    cfg = grid(32, 1)
    P = scene_hologram(gpu_ctx, cfg, 7, 6)
    res = api.convert_phase_only(P, cfg, 60, ctx=gpu_ctx)
    assert api.phase_only_loss(P, np.angle(P), cfg, ctx=gpu_ctx) == res.trace[0]
    assert api.phase_only_loss(P, res.hologram.phase, cfg, ctx=gpu_ctx) <= res.trace[0]


def test_gradient_matches_central_differences(gpu_ctx):
    """test_phase_only.cpp:103-131."""
    cfg = grid(32, 2)
    P = scene_hologram(gpu_ctx, cfg, 5, 6)
    theta = perturbed_arg(P, 3)
    _, g = api.phase_only_loss(P, theta, cfg, PhaseOnlyOptions(), want_grad=True, ctx=gpu_ctx)
    g = g.ravel()
    idx = list(range(0, theta.size, 97))
    fd = api.phase_gradient_oracle(P, theta, cfg, idx, 1e-5, ctx=gpu_ctx)
    healthy = 0.0
    for i in idx:
        healthy = max(healthy, abs(g[i]))
        rel = abs(g[i] - fd[i]) / max(abs(g[i]), abs(fd[i]), 1e-7)
        assert rel < 1e-4, (i, g[i], fd[i])
    assert healthy > 1e-6
    sparse = api.phase_gradient_oracle(P, theta, cfg, [idx[1], idx[3]], 1e-5, ctx=gpu_ctx)
    assert np.count_nonzero(sparse) == 2


def test_conjugation_flips_gradient(gpu_ctx):
    """test_phase_only.cpp:133-170."""
    cfg = grid(32, 2)
    P = scene_hologram(gpu_ctx, cfg, 5, 6)
    theta = perturbed_arg(P, 9)
    opt = PhaseOnlyOptions(lambda_ssim=0.0, prop=PropagationOptions(pad2x=False))
    l1, g = api.phase_only_loss(P, theta, cfg, opt, want_grad=True, ctx=gpu_ctx)
    l2, gc = api.phase_only_loss(np.conj(P), -theta, cfg, opt, want_grad=True, ctx=gpu_ctx)
    assert abs(l1 - l2) <= 1e-12 * abs(l1)
    rel = np.abs(g + gc) / np.maximum(np.maximum(np.abs(g), np.abs(gc)), 1e-8)
    assert rel.max() < 1e-6


def test_bad_inputs(gpu_ctx):
    """test_phase_only.cpp:172-199."""
    cfg = grid(32, 2)
    P = scene_hologram(gpu_ctx, cfg, 5, 4)
    theta = np.angle(P)
    big = grid(128, 2)
    with pytest.raises(HoloError):
        api.phase_gradient_oracle(np.zeros((3, 128, 128), complex), np.zeros((3, 128, 128)), big, ctx=gpu_ctx)
    flat = grid(32, 0)
    with pytest.raises(HoloError):
        api.phase_gradient_oracle(P, theta, flat, ctx=gpu_ctx)
    with pytest.raises(HoloError):
        api.convert_phase_only(P, flat, 1, ctx=gpu_ctx)
    with pytest.raises(HoloError):
        api.phase_only_loss(P, np.zeros(3), cfg, ctx=gpu_ctx)
    with pytest.raises(HoloError):
        api.phase_gradient_oracle(P, theta, cfg, [theta.size], ctx=gpu_ctx)
    with pytest.raises(HoloError):
        api.phase_gradient_oracle(P, theta, cfg, [], 0.0, ctx=gpu_ctx)
    with pytest.raises(HoloError):
        api.convert_phase_only(P, cfg, -1, ctx=gpu_ctx)
    with pytest.raises(HoloError):
        api.convert_phase_only(P, cfg, 1, 0.0, ctx=gpu_ctx)
    bad = P.copy()
    bad.flat[5] = np.nan
    with pytest.raises(HoloError) as e:
        api.convert_phase_only(bad, cfg, 1, ctx=gpu_ctx)
    assert e.value.kind == "numeric"


# ------------------------------------------------------------------ parity with the reference build

CASES = {
    "rgb_pad": (grid(32, 2), PhaseOnlyOptions()),
    "rgb_nopad": (grid(32, 2), PhaseOnlyOptions(prop=PropagationOptions(pad2x=False))),
    "mono_3planes": (grid(40, 3, (515e-9,)), PhaseOnlyOptions(lambda_ssim=0.3)),
    "no_ssim_local": (grid(24, 2), PhaseOnlyOptions(lambda_ssim=0.0,
                                                    prop=PropagationOptions(pad2x=True, local_band_limit=True))),
    "rect": (WaveConfig(nx=48, ny=36, num_planes=2), PhaseOnlyOptions()),
}


def case_inputs(ctx, name):
    cfg, opt = CASES[name]
    rgb = WaveConfig(nx=cfg.nx, ny=cfg.ny, num_planes=cfg.num_planes)
    P = scene_hologram(ctx, rgb, 5, 6)[: cfg.channels()]
    return cfg, opt, P


@pytest.mark.parametrize("name", sorted(CASES))
def test_loss_and_gradient_match_reference(gpu_ctx, ref, name):
    cfg, opt, P = case_inputs(gpu_ctx, name)
    theta = perturbed_arg(P, 4)
    loss, g = api.phase_only_loss(P, theta, cfg, opt, want_grad=True, ctx=gpu_ctx)
    rl, rg = ref.phase_only_loss(P, theta, cfg, opt.lambda_ssim, opt.prop, opt.use_adam)
    assert abs(loss - rl) <= 1e-10 * abs(rl), (loss, rl)
    assert rel_l2(g, rg) <= 1e-10, rel_l2(g, rg)


@pytest.mark.parametrize("name,adam", [("rgb_pad", False), ("rgb_nopad", False), ("mono_3planes", True)])
def test_conversion_trace_matches_reference(gpu_ctx, ref, name, adam):
    cfg, opt, P = case_inputs(gpu_ctx, name)
    opt.use_adam = adam
    res = api.convert_phase_only(P, cfg, 25, 0.05, opt, ctx=gpu_ctx)
    rphase, rtrace = ref.convert_phase_only(P, cfg, 25, 0.05, opt.lambda_ssim, opt.prop, adam)
    tr = np.asarray(res.trace)
    assert np.allclose(tr, rtrace, rtol=1e-8, atol=0), np.max(np.abs(tr - rtrace) / np.abs(rtrace))
    assert np.max(np.abs(res.hologram.phase - rphase)) <= 1e-7
