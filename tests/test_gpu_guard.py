"""Out-of-bounds write detection with guard bands (holo_ctx_set_guard /
holo_ctx_check_guards): compute-sanitizer is disabled on this GPU pool, so every
kernel family runs on small workloads with a 4 KB guard band after each scratch
buffer at its exact requested size, and the bands must come back intact.  The
negative test proves the check sees a write one byte past a buffer."""
import numpy as np
import pytest

from paper_2506_08350_b200 import _lib as L
from paper_2506_08350_b200 import api
from paper_2506_08350_b200.holotypes import PipelineOptions, PropagationOptions, WaveConfig
from paper_2506_08350_b200.scenes import front_camera, synthetic_scene

pytestmark = pytest.mark.gpu
RGB = (639e-9, 532e-9, 473e-9)


def _guarded_ctx(**kw):
    ctx = api.Context(0, **kw)
    ctx.set_guard(True)
    return ctx


def test_guard_detects_a_write_past_a_buffer():
    import torch

    ctx = _guarded_ctx()
    cfg = WaveConfig(nx=64, ny=64, wavelengths=RGB, num_planes=2)
    ctx.upload_scene(synthetic_scene(500, cfg, 1))
    ctx.render(front_camera(cfg), cfg, outputs=L.OUT_LAYERS | L.OUT_HOLOGRAM)
    ctx.check_guards()
    ptr, nbytes = ctx.buffer(L.BUF_LAYERS)
    torch.as_tensor(api._CudaArray(ptr + nbytes, (1,), "|u1"), device="cuda").zero_()
    with pytest.raises(L.HoloError) as e:
        ctx.check_guards()
    assert "layers" in str(e.value)


@pytest.mark.parametrize("W,H", [(128, 128), (96, 80)])
def test_forward_and_every_sort_path_stay_in_bounds(W, H):
    ctx = _guarded_ctx()
    cfg = WaveConfig(nx=W, ny=H, wavelengths=RGB, num_planes=2)
    s = synthetic_scene(12000, cfg, 32)
    s.positions[:4000, :2] *= 0.03   # buckets above 1024 entries
    s.positions[4000:8000, :2] *= 0.4
    g = api.pipeline_forward(s, front_camera(cfg), cfg, ctx=ctx)
    sizes = np.diff(g.raster.bucket_start.astype(np.int64))
    assert sizes.max() > 1024 and ((sizes > 256) & (sizes <= 1024)).any()
    api.pipeline_forward(synthetic_scene(800, cfg, 3), front_camera(cfg), cfg,
                         PipelineOptions(prop=PropagationOptions(pad2x=True)), ctx=ctx)
    ctx.check_guards()


def test_overflowed_async_frame_stays_in_bounds():
    """The ADVICE case: an asynchronous frame far over its reserved capacity with
    many buckets above the in-CTA sort capacity (k_find_large's list)."""
    cfg = WaveConfig(nx=64, ny=64, wavelengths=RGB, num_planes=2)
    s = synthetic_scene(20000, cfg, 4)
    s.positions[:, :2] *= 0.05
    ctx = _guarded_ctx(use_torch_stream=False)
    ctx.upload_scene(s)
    ctx.set_async(True)
    ctx.reserve_entries(100)
    ctx.render(front_camera(cfg), cfg, outputs=L.OUT_HOLOGRAM | L.OUT_INTENSITY | L.OUT_AUX | L.OUT_LISTS)
    with pytest.raises(L.HoloError):
        ctx.frame_status()
    ctx.check_guards()


def test_training_step_and_backward_stay_in_bounds():
    import torch

    ctx = _guarded_ctx()
    cfg = WaveConfig(nx=64, ny=48, wavelengths=RGB, num_planes=3)
    s = synthetic_scene(600, cfg, 5)
    cam = front_camera(cfg)
    ctx.upload_scene(s)
    ctx.render(cam, cfg, outputs=L.OUT_INTENSITY)
    ints = ctx.download(L.BUF_INTENSITY, np.float32, (3, 3, 48, 64))
    targets = torch.from_numpy(0.9 * ints.astype(np.float64)).to("cuda:0")
    masks = torch.zeros((3, 48, 64), dtype=torch.float64, device="cuda:0")
    _, grads = ctx.total_loss(cam, cfg, targets, masks, n=s.size())
    assert api.Optimizer(ctx).step(grads)
    ctx.render(cam, cfg, outputs=L.OUT_LAYERS | L.OUT_AUX)
    ctx.raster_backward(cam, cfg, None, torch.ones((3, 3, 48, 64), dtype=torch.complex64, device="cuda:0"),
                        s.size())
    u = np.random.default_rng(0).standard_normal((3, 48, 64)) + 0j
    for prec in ("f32", "f64"):
        ctx.propagate(u, cfg, 1e-3, precision=prec)
    api.phase_only_loss(np.exp(1j * u), np.zeros((3, 48, 64)), cfg, ctx=ctx)
    ctx.check_guards()


def test_group_sharded_path_stays_in_bounds():
    ctx = _guarded_ctx()
    cfg = WaveConfig(nx=128, ny=128, wavelengths=RGB, num_planes=4)
    g = api.Group(ctx)
    g.set_lanes(2)
    g.upload_scene(synthetic_scene(5000, cfg, 6))
    g.render([front_camera(cfg)] * 3, cfg, flags=L.GROUP_SHARDED_PATH | L.GROUP_GATHER_HOLOGRAM)
    g.synchronize()
    ctx.check_guards()
    g.close()
