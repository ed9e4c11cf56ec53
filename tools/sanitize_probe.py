"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck) over
every kernel family of libholo_cuda: the forward render on static and
runtime-planned grids, all three bucket sorts, an overflowed asynchronous frame
(the large-bucket list bounded by the clamped capacity), the raster and pipeline
backward, a training step, phase-only loss, the f32/f64 operators and the group
renderer's per-channel sharded path.

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_probe.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200 import api  # noqa: E402
from paper_2506_08350_b200.holotypes import PipelineOptions, PropagationOptions, WaveConfig  # noqa: E402
from paper_2506_08350_b200.scenes import front_camera, synthetic_scene  # noqa: E402

RGB = (639e-9, 532e-9, 473e-9)


def main():
    ctx = api.Context(0)
    # forward: static plans (128^2) and runtime plans (96 x 80), all raster outputs
    for (W, H) in ((128, 128), (96, 80)):
        cfg = WaveConfig(nx=W, ny=H, wavelengths=RGB, num_planes=3)
        s = synthetic_scene(4000, cfg, 1)
        s.positions[:1500, :2] *= 0.03  # buckets above 1024 entries (device-wide sort)
        s.positions[1500:2500, :2] *= 0.4
        api.pipeline_forward(s, front_camera(cfg), cfg, ctx=ctx)
    # pad2x operators
    cfg = WaveConfig(nx=64, ny=48, wavelengths=RGB, num_planes=2)
    s = synthetic_scene(800, cfg, 2)
    api.pipeline_forward(s, front_camera(cfg), cfg, PipelineOptions(prop=PropagationOptions(pad2x=True)), ctx=ctx)
    # overflowed asynchronous frame with large buckets
    cfg = WaveConfig(nx=64, ny=64, wavelengths=RGB, num_planes=2)
    s = synthetic_scene(8000, cfg, 3)
    s.positions[:, :2] *= 0.05
    c2 = api.Context(0, use_torch_stream=False)
    c2.upload_scene(s)
    c2.set_async(True)
    c2.reserve_entries(100)
    c2.render(front_camera(cfg), cfg, outputs=L.OUT_HOLOGRAM | L.OUT_INTENSITY | L.OUT_AUX)
    try:
        c2.frame_status()
    except L.HoloError:
        pass
    c2.close()
    # backward and one training step
    cfg = WaveConfig(nx=64, ny=48, wavelengths=RGB, num_planes=3)
    s = synthetic_scene(600, cfg, 4)
    cam = front_camera(cfg)
    ctx.upload_scene(s)
    ctx.render(cam, cfg, outputs=L.OUT_INTENSITY | L.OUT_REPLAYED | L.OUT_AUX)
    ints = ctx.download(L.BUF_INTENSITY, np.float32, (3, 3, 48, 64))
    targets = torch.from_numpy(0.9 * ints.astype(np.float64)).to("cuda:0")
    masks = torch.zeros((3, 48, 64), dtype=torch.float64, device="cuda:0")
    _, grads = ctx.total_loss(cam, cfg, targets, masks, n=s.size())
    opt = api.Optimizer(ctx)
    opt.step(grads)
    ctx.render(cam, cfg, outputs=L.OUT_LAYERS | L.OUT_AUX)
    gl = torch.ones((3, 3, 48, 64), dtype=torch.complex64, device="cuda:0")
    ctx.raster_backward(cam, cfg, None, gl, s.size())
    # operators (f32 / f64) and phase-only
    u = np.random.default_rng(0).standard_normal((3, 48, 64)) + 0j
    for prec in ("f32", "f64"):
        ctx.propagate(u, cfg, 1e-3, precision=prec)
        ctx.fft2(u, precision=prec)
    api.phase_only_loss(np.exp(1j * u), np.zeros((3, 48, 64)), cfg, ctx=ctx)
    # group renderer: per-channel sharded path (world 1, NCCL communicator of one)
    cfg = WaveConfig(nx=128, ny=128, wavelengths=RGB, num_planes=4)
    g = api.Group(ctx)
    g.upload_scene(synthetic_scene(5000, cfg, 5))
    g.render([front_camera(cfg)], cfg, flags=L.GROUP_SHARDED_PATH | L.GROUP_GATHER_HOLOGRAM)
    g.synchronize()
    g.close()
    ctx.synchronize()
    torch.cuda.synchronize()
    print("sanitize_probe: done")


if __name__ == "__main__":
    main()
