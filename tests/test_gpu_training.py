"""GPU training step against the reference: the loss terms (losses.cpp, ssim.cpp),
total_loss (pipeline.cpp:30-95) and optimizer_step (optimizer.cpp:102-133).

Bars:
* losses on given f64 stacks: f64 on the GPU in the reference's operation order
  (row sums folded like fold_partials, no FMA contraction) -- values and dL/dI
  within 1e-12 relative of the reference build (in practice equal);
* total_loss: the render computes in fp32 (the north star's precision), so the
  loss terms agree to 1e-5 relative, PSNR to 1e-4 dB, gradients to rel-L2 1e-3
  (the backward tests' bar) and the opacity term to 1e-12;
* optimizer: f64, same operation order -> parameters within 1e-13 relative.
The reference's own KATs (tests/test_losses.cpp, test_optimizer.cpp) run on the
GPU path too."""
import numpy as np
import pytest

from conftest import desk_config, front_camera, random_scene, rel_l2
from oracle.oracle import Oracle
from paper_2506_08350_b200 import api
from paper_2506_08350_b200._lib import HoloError
from paper_2506_08350_b200.holotypes import OptimizerConfig, PipelineOptions, RenderSettings

pytestmark = pytest.mark.gpu

GROUPS = ("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases", "plane_logits")


@pytest.fixture(scope="module")
def ref():
    if not Oracle.available("ref"):
        pytest.skip("reference build (oracle/_ref) not available")
    return Oracle("ref")


def torch_dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda:0")


def stacks(L, C, H, W, seed):
    rng = np.random.default_rng(seed)
    I = rng.random((L, C, H, W))
    G = np.clip(I + 0.2 * rng.standard_normal((L, C, H, W)), 0.0, 1.0)
    M = (rng.random((L, H, W)) > 0.5).astype(np.float64)
    return I, G, M


def close(a, b, tol):
    return abs(a - b) <= tol * max(abs(a), abs(b), 1e-300)


# ------------------------------------------------------------------ loss terms on given stacks

@pytest.mark.parametrize("shape", [(2, 3, 20, 24), (1, 3, 11, 11), (3, 1, 37, 53), (2, 2, 64, 48)])
@pytest.mark.parametrize("plain", [False, True])
def test_losses_match_reference(gpu_ctx, ref, shape, plain):
    I, G, M = stacks(*shape, seed=sum(shape) + plain)
    opt = PipelineOptions(lambda_ssim=0.2, use_plain_mse=plain)
    b, g = api.losses(I, G, None if plain else M, opt, ctx=gpu_ctx)
    r, s, ps, rg = ref.losses(I, G, M, lambda_ssim=0.2, plain=plain)
    assert close(b.recon, r, 1e-12), (b.recon, r)
    assert close(b.ssim, s, 1e-12), (b.ssim, s)
    assert np.allclose(b.psnr, ps, rtol=1e-12, atol=0)
    assert b.opacity == 0.0 and close(b.total, r + s, 1e-12)
    assert rel_l2(g, rg) <= 1e-12, rel_l2(g, rg)


def test_losses_bit_pattern(gpu_ctx, ref):
    """The fold order is the reference's: values equal, not just close."""
    I, G, M = stacks(2, 3, 32, 40, 5)
    b, g = api.losses(I, G, M, PipelineOptions(lambda_ssim=0.005), ctx=gpu_ctx)
    r, s, ps, rg = ref.losses(I, G, M, lambda_ssim=0.005)
    assert b.recon == r
    assert np.array_equal(np.asarray(b.psnr), ps)
    # the SSIM blur order matches too; allow the last bit in case a libm differs
    assert close(b.ssim, s, 4e-16)
    assert np.max(np.abs(g - rg)) <= 4e-16 * np.max(np.abs(rg))


def test_ssim_identity_and_kats(gpu_ctx):
    """test_losses.cpp:65-110: ssim(a, a) = 1 (loss term 0), contrast inversion < 0.2."""
    rng = np.random.default_rng(3)
    a = rng.random((1, 2, 16, 24))
    b, _ = api.losses(a, a, None, PipelineOptions(lambda_ssim=1.0, use_plain_mse=True), ctx=gpu_ctx)
    assert abs(b.ssim) <= 1e-12 and b.recon == 0.0 and b.psnr == [99.0]
    x = np.zeros((1, 1, 32, 32))
    for y in range(32):
        for px in range(32):
            x[0, 0, y, px] = 1.0 if (y // 4 + px // 4) % 2 else 0.0
    b, _ = api.losses(x, 1.0 - x, None, PipelineOptions(lambda_ssim=1.0, use_plain_mse=True), ctx=gpu_ctx)
    s = 1.0 - b.ssim
    assert -1.0 <= s < 0.2


def test_loss_kats(gpu_ctx):
    """test_losses.cpp:118-203: MSE over planes, the hand-computed masked term, psnr."""
    rng = np.random.default_rng(1)
    gt = rng.random((2, 3, 8, 8))
    off = gt + 0.1
    no_ssim = PipelineOptions(lambda_ssim=0.0, use_plain_mse=True)
    b, _ = api.losses(off, gt, None, no_ssim, ctx=gpu_ctx)
    assert close(b.recon, 0.01, 1e-12)
    assert np.allclose(b.psnr, 20.0, rtol=1e-12)
    b, _ = api.losses(gt, gt, None, no_ssim, ctx=gpu_ctx)
    assert b.recon == 0.0 and b.psnr == [99.0, 99.0]
    masked = PipelineOptions(lambda_ssim=0.0)
    one = lambda v: np.full((1, 1, 1, 1), v)  # noqa: E731
    b, _ = api.losses(one(0.5), one(1.0), np.ones((1, 1, 1)), masked, ctx=gpu_ctx)
    assert close(b.recon, 0.75, 1e-14)
    b, _ = api.losses(one(0.5), one(1.0), np.zeros((1, 1, 1)), masked, ctx=gpu_ctx)
    assert close(b.recon, 0.5, 1e-14)


def test_loss_gradient_finite_differences(gpu_ctx):
    """test_losses.cpp:96-110, 150-171: dL/dI of recon + ssim against central differences."""
    I, G, M = stacks(2, 1, 16, 14, 21)
    opt = PipelineOptions(lambda_ssim=0.5)
    _, g = api.losses(I, G, M, opt, ctx=gpu_ctx)
    rng = np.random.default_rng(0)
    h = 1e-6
    for _ in range(12):
        idx = tuple(int(rng.integers(0, s)) for s in I.shape)
        Ip, Im = I.copy(), I.copy()
        Ip[idx] += h
        Im[idx] -= h
        fd = (api.losses(Ip, G, M, opt, ctx=gpu_ctx)[0].total - api.losses(Im, G, M, opt, ctx=gpu_ctx)[0].total) / (2 * h)
        assert abs(g[idx] - fd) <= 1e-6 * max(abs(fd), abs(g[idx])) + 1e-10, (idx, g[idx], fd)


def test_loss_errors(gpu_ctx):
    I, G, M = stacks(1, 1, 8, 16, 2)
    with pytest.raises(HoloError) as e:
        api.losses(I, G, M, PipelineOptions(lambda_ssim=0.005), ctx=gpu_ctx)  # ssim.cpp:71-72
    assert e.value.kind == "config"
    with pytest.raises(HoloError) as e:
        api.losses(I, G, None, PipelineOptions(lambda_ssim=0.0), ctx=gpu_ctx)
    assert e.value.kind == "usage"


# ------------------------------------------------------------------ total_loss

def loss_case(case):
    cfg = desk_config(48, 2)
    cam = front_camera(cfg)
    scene = random_scene(40, cfg, 61)
    opt = PipelineOptions(lambda_ssim=0.05, lambda_opacity=1e-2)
    if case == "plain":
        opt.use_plain_mse = True
    elif case == "soft":
        opt.raster = RenderSettings(soft_assignment=True)
    rng = np.random.default_rng(7)
    targets = rng.random((cfg.num_planes, 3, cfg.ny, cfg.nx)) * 0.5
    masks = (rng.random((cfg.num_planes, cfg.ny, cfg.nx)) > 0.6).astype(np.float64)
    return cfg, cam, scene, opt, targets, masks


@pytest.mark.parametrize("case", ["default", "plain", "soft"])
def test_total_loss_matches_reference(gpu_ctx, ref, case):
    cfg, cam, scene, opt, targets, masks = loss_case(case)
    b, g = api.total_loss(scene, cam, cfg, targets, masks, opt, ctx=gpu_ctx)
    rb, rps, rg = ref.total_loss(scene, cam, cfg, opt.raster, opt.prop, targets, masks, lambda_ssim=opt.lambda_ssim,
                                 lambda_opacity=opt.lambda_opacity, plain=opt.use_plain_mse)
    assert close(b.recon, rb["recon"], 1e-5), (b.recon, rb)
    assert close(b.ssim, rb["ssim"], 1e-5), (b.ssim, rb)
    assert close(b.opacity, rb["opacity"], 1e-12), (b.opacity, rb)
    assert close(b.total, rb["total"], 1e-5)
    assert np.allclose(b.psnr, rps, atol=1e-4, rtol=0)
    assert abs(b.psnr_mean - rb["psnr_mean"]) <= 1e-4
    errs = {k: rel_l2(g[k], rg[k]) for k in GROUPS + ("mu_screen",) if np.abs(rg[k]).max() > 0}
    assert all(e <= 1e-3 for e in errs.values()), errs


def test_total_loss_without_grads(gpu_ctx, ref):
    cfg, cam, scene, opt, targets, masks = loss_case("default")
    b, g = api.total_loss(scene, cam, cfg, targets, masks, opt, want_grads=False, ctx=gpu_ctx)
    assert g is None
    rb, _, _ = ref.total_loss(scene, cam, cfg, opt.raster, opt.prop, targets, masks, lambda_ssim=opt.lambda_ssim,
                              lambda_opacity=opt.lambda_opacity, grads=False)
    assert close(b.total, rb["total"], 1e-5)


# ------------------------------------------------------------------ optimizer

REF_CFG_KEYS = ("lr_positions", "lr_rotations", "lr_log_scales", "lr_amplitudes", "lr_phases", "lr_opacities",
                "lr_plane_logits", "beta1", "beta2", "beta3", "eps", "lr_floor")


def random_grads(scene, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    return {k: scale * rng.standard_normal(np.shape(getattr(scene, k))) for k in GROUPS}


@pytest.mark.parametrize("adam", [False, True])
def test_optimizer_matches_reference(gpu_ctx, ref, adam):
    cfg = desk_config(48, 3)
    scene = random_scene(50, cfg, 5)
    oc = OptimizerConfig(use_adam=adam, schedule_total=3)  # the cosine reaches its floor inside the run
    steps = [random_grads(scene, s) for s in range(5)]
    steps[2] = dict(steps[2])
    steps[2]["phases"] = steps[2]["phases"].copy()
    steps[2]["phases"][3, 1] = np.inf  # a skipped step (optimizer.cpp:110-115)
    gpu_ctx.upload_scene(scene)
    opt = api.Optimizer(gpu_ctx)
    applied = []
    for g in steps:
        applied.append(opt.step({k: torch_dev(v) for k, v in g.items()}, oc))
    assert applied == [True, True, False, True, True]
    assert opt.counts() == (4, 1)
    out = gpu_ctx.download_scene(scene.size(), scene.num_planes)
    want, ref_applied = ref.optimizer_run(scene, steps, [getattr(oc, k) for k in REF_CFG_KEYS], use_adam=adam,
                                          schedule_total=oc.schedule_total)
    assert list(ref_applied) == [1, 1, 0, 1, 1]
    for k in GROUPS:
        got = np.ravel(getattr(out, k))
        assert np.allclose(got, want[k], rtol=1e-13, atol=1e-15), (k, np.max(np.abs(got - want[k])))
    opt.close()


def test_optimizer_zero_gradients_and_renormalize(gpu_ctx):
    """test_optimizer.cpp:83-112: zero gradients leave the parameters untouched."""
    cfg = desk_config(32, 2)
    scene = random_scene(20, cfg, 9)
    scene.rotations = scene.rotations / np.linalg.norm(scene.rotations, axis=1, keepdims=True)
    gpu_ctx.upload_scene(scene)
    opt = api.Optimizer(gpu_ctx)
    zero = {k: torch_dev(np.zeros(np.shape(getattr(scene, k)))) for k in GROUPS}
    assert opt.step(zero)
    out = gpu_ctx.download_scene(scene.size(), scene.num_planes)
    for k in GROUPS:
        assert np.allclose(getattr(out, k), getattr(scene, k), rtol=0, atol=1e-15), k


def test_training_loop_lowers_the_loss(gpu_ctx):
    """A few total_loss -> optimizer_step iterations on the resident scene (the
    trainer's inner loop, trainer.cpp) fit a target rendered from a perturbed scene."""
    cfg = desk_config(48, 2)
    cam = front_camera(cfg)
    truth = random_scene(40, cfg, 61)
    opt = PipelineOptions()
    target = api.pipeline_forward(truth, cam, cfg, opt, ctx=gpu_ctx, raster=False, replayed=False).intensities
    target = torch_dev(np.stack(target))
    masks = torch_dev(np.zeros((2, 48, 48)))
    start = random_scene(40, cfg, 61)
    start.positions = start.positions + 2e-4 * np.random.default_rng(0).standard_normal(start.positions.shape)
    start.amplitudes = start.amplitudes * 0.7
    gpu_ctx.upload_scene(start)
    optim = api.Optimizer(gpu_ctx)
    oc = OptimizerConfig(lr_amplitudes=0.02)
    losses = []
    for _ in range(15):
        b, g = gpu_ctx.total_loss(cam, cfg, target, masks, opt, n=start.size())
        losses.append(b.total)
        assert optim.step(g, oc)
    assert losses[-1] < 0.7 * losses[0], losses


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_self_target_full_size(gpu_ctx, name):
    """test_pipeline.cpp:93-113 at BASELINE sizes (a size-independent property):
    a scene rendered against its own intensities has zero reconstruction loss,
    PSNR 99 dB and vanishing gradients."""
    import torch

    from paper_2506_08350_b200 import _lib as L
    from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene

    c = CONFIGS[name]
    cfg, cam = c.wave(), c.cameras()[0]
    scene = synthetic_scene(c.n, cfg, c.seed)
    gpu_ctx.upload_scene(scene)
    gpu_ctx.render(cam, cfg, outputs=L.OUT_REPLAYED)
    Cn, H, W = cfg.channels(), cfg.ny, cfg.nx
    rep = gpu_ctx.tensor(L.BUF_REPLAYED, "c8", (cfg.num_planes, Cn, H, W)).to(torch.complex128)
    target = (rep.real ** 2 + rep.imag ** 2).contiguous()  # |replay|^2 in f64, as total_loss forms it
    masks = torch.zeros((cfg.num_planes, H, W), dtype=torch.float64, device="cuda:0")
    opt = PipelineOptions(lambda_opacity=0.0)
    b, g = gpu_ctx.total_loss(cam, cfg, target, masks, opt, n=scene.size())
    assert b.recon == 0.0 and b.psnr_mean == 99.0 and abs(b.ssim) < 1e-12
    worst = max(float(v.abs().max()) for k, v in g.items() if k != "mu_screen")
    assert worst < 1e-8, worst


def test_optimizer_rejects_a_resized_scene(gpu_ctx):
    """optimizer.cpp:105-108: moment buffers sized for one scene do not take another
    (densification: create a fresh optimizer state)."""
    cfg = desk_config(32, 2)
    a, b = random_scene(20, cfg, 1), random_scene(30, cfg, 2)
    gpu_ctx.upload_scene(a)
    opt = api.Optimizer(gpu_ctx)
    assert opt.step({k: torch_dev(np.zeros(np.shape(getattr(a, k)))) for k in GROUPS})
    gpu_ctx.upload_scene(b)
    with pytest.raises(HoloError) as e:
        opt.step({k: torch_dev(np.zeros(np.shape(getattr(b, k)))) for k in GROUPS})
    assert e.value.kind == "config"
    fresh = api.Optimizer(gpu_ctx)
    assert fresh.step({k: torch_dev(np.zeros(np.shape(getattr(b, k)))) for k in GROUPS})
    assert fresh.counts() == (1, 0)


def test_total_loss_rejects_bad_inputs(gpu_ctx):
    cfg, cam, scene, opt, targets, masks = loss_case("default")
    with pytest.raises(HoloError):  # masks required unless plain MSE
        api.total_loss(scene, cam, cfg, targets, None, opt, ctx=gpu_ctx)
    small = desk_config(8, 2)  # SSIM needs >= 11 pixels (ssim.cpp:71-72)
    with pytest.raises(HoloError) as e:
        api.total_loss(random_scene(5, small, 3), front_camera(small), small, np.zeros((2, 3, 8, 8)),
                       np.zeros((2, 8, 8)), opt, ctx=gpu_ctx)
    assert e.value.kind == "config"
