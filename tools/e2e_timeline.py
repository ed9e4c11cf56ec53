"""Timeline of the single-context end-to-end pipeline: when each frame's scene
upload, render and downloads finish on the copy-in, compute and copy-out streams."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200.api import Context  # noqa: E402
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene  # noqa: E402

c = CONFIGS["C3"]
wave, cam = c.wave(), c.cameras()[0]
scene = synthetic_scene(c.n, wave, c.seed)
pinned = [torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).pin_memory() for a in
          (scene.positions, scene.rotations, scene.log_scales, scene.amplitudes, scene.opacity_logits, scene.phases,
           scene.plane_logits)]
ptrs = [p.data_ptr() for p in pinned]
Cn, H, W, Lp = wave.channels(), wave.ny, wave.nx, wave.num_planes
hh = torch.empty(Cn * H * W * 2, dtype=torch.float32).pin_memory()
ih = torch.empty(Lp * Cn * H * W, dtype=torch.float32).pin_memory()
ctx = Context(0, use_torch_stream=False)
s_in, s_comp, s_out = (torch.cuda.ExternalStream(x) for x in (ctx.copy_stream(0), ctx.stream(), ctx.copy_stream(1)))
outs = L.OUT_HOLOGRAM | L.OUT_INTENSITY
ctx.upload_scene_pointers(c.n, Lp, ptrs, device=False)
ctx.render(cam, wave, None, None, outputs=outs)
ctx.synchronize()
ctx.set_async(True)
N = 14
E = {k: [torch.cuda.Event(enable_timing=True) for _ in range(N)] for k in ("up", "r", "d")}
base = torch.cuda.Event(enable_timing=True)
for i in range(3):
    ctx.upload_scene_pointers(c.n, Lp, ptrs, device=False)
    ctx.render(cam, wave, None, None, outputs=outs)
    ctx.download_into(L.BUF_HOLOGRAM, hh.data_ptr(), hh.numel() * 4, wait=False)
    ctx.download_into(L.BUF_INTENSITY, ih.data_ptr(), ih.numel() * 4, wait=False)
ctx.synchronize()
base.record(s_comp)
for i in range(N):
    ctx.upload_scene_pointers(c.n, Lp, ptrs, device=False)
    E["up"][i].record(s_in)
    ctx.render(cam, wave, None, None, outputs=outs)
    E["r"][i].record(s_comp)
    ctx.download_into(L.BUF_HOLOGRAM, hh.data_ptr(), hh.numel() * 4, wait=False)
    ctx.download_into(L.BUF_INTENSITY, ih.data_ptr(), ih.numel() * 4, wait=False)
    E["d"][i].record(s_out)
ctx.synchronize()
torch.cuda.synchronize()
prev = None
for i in range(N):
    t = [base.elapsed_time(E[k][i]) for k in ("up", "r", "d")]
    dd = "" if prev is None else f"   (+{t[0] - prev[0]:.2f} +{t[1] - prev[1]:.2f} +{t[2] - prev[2]:.2f})"
    print(f"frame {i:2d}: upload done {t[0]:7.2f}  render done {t[1]:7.2f}  download done {t[2]:7.2f}{dd}")
    prev = t
ctx.frame_status()
