"""Where does the end-to-end frame time go?  Frames rotate over K contexts, each
step doing a subset of {scene upload (pinned), render, result download (pinned)}."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200.api import Context  # noqa: E402
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene  # noqa: E402

c = CONFIGS["C3"]
wave, cam = c.wave(), c.cameras()[0]
scene = synthetic_scene(c.n, wave, c.seed)
arrays = [np.ascontiguousarray(a, dtype=np.float64) for a in
          (scene.positions, scene.rotations, scene.log_scales, scene.amplitudes, scene.opacity_logits, scene.phases,
           scene.plane_logits)]
pinned = [torch.from_numpy(a).pin_memory() for a in arrays]
ptrs = [p.data_ptr() for p in pinned]
Cn, H, W, Lp = wave.channels(), wave.ny, wave.nx, wave.num_planes
outs = L.OUT_HOLOGRAM | L.OUT_INTENSITY


def probe(K, up, rend, down, n=20):
    ctxs = [Context(0, use_torch_stream=False) for _ in range(K)]
    hb = [(torch.empty(Cn * H * W * 2, dtype=torch.float32).pin_memory(),
           torch.empty(Lp * Cn * H * W, dtype=torch.float32).pin_memory()) for _ in range(K)]
    for cx in ctxs:
        cx.upload_scene_pointers(c.n, Lp, ptrs, device=False)
        cx.render(cam, wave, None, None, outputs=outs)
        cx.synchronize()
        cx.set_async(True)

    def step(i):
        cx = ctxs[i % K]
        hh, ih = hb[i % K]
        if up:
            cx.upload_scene_pointers(c.n, Lp, ptrs, device=False)
        if rend:
            cx.render(cam, wave, None, None, outputs=outs)
        if down:
            cx.download_into(L.BUF_HOLOGRAM, hh.data_ptr(), hh.numel() * 4, wait=False)
            cx.download_into(L.BUF_INTENSITY, ih.data_ptr(), ih.numel() * 4, wait=False)

    for i in range(K):
        step(i)
    for cx in ctxs:
        cx.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        step(i)
    th = time.perf_counter() - t0
    for cx in ctxs:
        cx.synchronize()
    dt = time.perf_counter() - t0
    for cx in ctxs:
        cx.frame_status()
        cx.close()
    print(f"K={K} up={up} render={rend} down={down}: {dt / n * 1e3:6.2f} ms/frame (host enqueue {th / n * 1e3:.2f})",
          flush=True)


for K in (1, 3):
    for flags in ((1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (0, 1, 1), (1, 0, 1), (1, 1, 1)):
        probe(K, *flags)
