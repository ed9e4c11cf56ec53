"""GPU gradients against the reference build (oracle/_ref): raster_backward
(rasterizer.cpp:332-528) and the gradient branch of total_loss
(pipeline.cpp:63-80).

Bars: every scene-gradient array within rel-L2 1e-3 of the reference's f64
result (the GPU sweeps pixels in fp32 -- the forward's own precision -- and
merges / chains per Gaussian in f64); grad_layers / grad_hologram of the adjoint
propagation within rel-L2 1e-4 (fp32 fields, as the forward)."""
import numpy as np
import pytest

from conftest import desk_config, front_camera, mild_posed_camera, random_scene, rel_l2
from oracle.oracle import Oracle
from paper_2506_08350_b200 import _lib as L
from paper_2506_08350_b200 import api
from paper_2506_08350_b200._lib import HoloError
from paper_2506_08350_b200.holotypes import PipelineOptions, PropagationOptions, RenderSettings, WaveConfig
from paper_2506_08350_b200.scenes import front_camera as wide_camera
from paper_2506_08350_b200.scenes import synthetic_scene

pytestmark = pytest.mark.gpu
RGB = (639e-9, 532e-9, 473e-9)
GRAD_TOL = 1e-3


@pytest.fixture(scope="module")
def ref():
    if not Oracle.available("ref"):
        pytest.skip("reference build (oracle/_ref) not available")
    return Oracle("ref")


def field(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def compare(g, r, tol=GRAD_TOL):
    errs = {}
    for k, v in r.items():
        if np.abs(v).max() == 0.0:
            assert np.abs(g[k]).max() <= 1e-12, k
            continue
        errs[k] = rel_l2(g[k], v)
    bad = {k: e for k, e in errs.items() if e > tol}
    assert not bad, (bad, errs)
    return errs


@pytest.mark.parametrize("case", ["gradcheck", "default", "posed", "soft", "tile8"])
def test_raster_backward_matches_reference(gpu_ctx, ref, case):
    cfg = desk_config(48, 2)
    cam = front_camera(cfg)
    st = RenderSettings()
    scene = random_scene(40, cfg, 61)
    if case == "gradcheck":  # helpers.hpp:105-111
        st = RenderSettings(alpha_floor=0.0, term_eps=0.0, radius_form_cap=80.0)
    elif case == "posed":
        cam = mild_posed_camera(cfg)
    elif case == "soft":
        st = RenderSettings(soft_assignment=True, soft_tau=1.0)
    elif case == "tile8":
        st = RenderSettings(tile=8)
    gl = field((cfg.num_planes, 3, cfg.ny, cfg.nx), 900)
    g = api.raster_backward(scene, cam, cfg, st, gl, ctx=gpu_ctx)
    r = ref.raster_backward(scene, cam, cfg, st, gl)
    compare(g, r)


def test_raster_backward_dense_scene(gpu_ctx, ref):
    # many overlapping splats per tile: long back-to-front sweeps
    cfg = WaveConfig(nx=128, ny=96, wavelengths=RGB, num_planes=3)
    scene = synthetic_scene(6000, cfg, 62)
    cam = wide_camera(cfg)
    gl = field((3, 3, 96, 128), 901)
    g = api.raster_backward(scene, cam, cfg, RenderSettings(), gl, ctx=gpu_ctx)
    r = ref.raster_backward(scene, cam, cfg, RenderSettings(), gl)
    compare(g, r)


@pytest.mark.parametrize("n,W,H,Lp,prop", [
    (300, 64, 48, 3, PropagationOptions()),
    (2000, 96, 80, 2, PropagationOptions()),                      # runtime-planned FFT sizes
    (300, 48, 32, 2, PropagationOptions(pad2x=True)),
    (300, 64, 48, 2, PropagationOptions(local_band_limit=True)),
])
def test_pipeline_backward_matches_reference(gpu_ctx, ref, n, W, H, Lp, prop):
    cfg = WaveConfig(nx=W, ny=H, wavelengths=RGB, num_planes=Lp)
    scene = synthetic_scene(n, cfg, 63)
    cam = wide_camera(cfg)
    gi = np.random.default_rng(7).standard_normal((Lp, 3, H, W))
    opt = PipelineOptions(prop=prop)
    g, gl, gh = api.pipeline_backward(scene, cam, cfg, opt, gi, ctx=gpu_ctx)
    r, rgh, rgl = ref.pipeline_backward(scene, cam, cfg, RenderSettings(), prop, gi)
    assert rel_l2(gh, rgh) < 1e-4
    assert rel_l2(gl, rgl) < 1e-4
    compare(g, r)


def test_backward_needs_the_forward_state(gpu_ctx):
    import torch

    cfg = desk_config(32, 2)
    cam = front_camera(cfg)
    s = random_scene(5, cfg, 3)
    gpu_ctx.upload_scene(s)
    gpu_ctx.render(cam, cfg, None, None, outputs=L.OUT_HOLOGRAM)  # no aux outputs
    gl = torch.zeros((2, 3, 32, 32), dtype=torch.complex64, device="cuda")
    with pytest.raises(HoloError) as e:
        gpu_ctx.raster_backward(cam, cfg, None, gl, s.size())
    assert e.value.kind == "usage"
    gpu_ctx.render(cam, cfg, None, None, outputs=L.OUT_AUX)
    other = front_camera(cfg, focal=120.0)
    with pytest.raises(HoloError) as e:
        gpu_ctx.raster_backward(other, cfg, None, gl, s.size())
    assert e.value.kind == "usage"
    gi = torch.zeros((2, 3, 32, 32), dtype=torch.float32, device="cuda")
    with pytest.raises(HoloError):  # no replayed fields in that render
        gpu_ctx.pipeline_backward(cam, cfg, None, None, gi, s.size())


def test_backward_is_bitwise_deterministic(gpu_ctx):
    """test_pipeline.cpp:262-288: gradients identical run to run (no float atomics
    in the per-entry reduction; the per-Gaussian merge is in a fixed order)."""
    cfg = desk_config(64, 3)
    cam = front_camera(cfg)
    scene = random_scene(300, cfg, 17)
    gi = np.random.default_rng(2).standard_normal((3, 3, 64, 64))
    runs = [api.pipeline_backward(scene, cam, cfg, PipelineOptions(), gi, ctx=gpu_ctx)[0] for _ in range(3)]
    for k in runs[0]:
        assert np.array_equal(runs[0][k], runs[1][k]) and np.array_equal(runs[0][k], runs[2][k]), k
