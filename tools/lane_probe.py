"""Per-frame host and device times of a plane-sharded rank (callback transport with
a no-op sum) with two lanes: looking for stalls."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200.api import Context, Group  # noqa: E402
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene  # noqa: E402

c = CONFIGS["C3"]
wave, cam = c.wave(), c.cameras()[0]
scene = synthetic_scene(c.n, wave, c.seed)
outs = L.OUT_INTENSITY | L.OUT_HOLOGRAM
world, lanes = int(sys.argv[1]), int(sys.argv[2])
ctx = Context(0)
g = Group(ctx, world, 0, world, allreduce=lambda *a: 0)
if lanes > 1:
    g.set_lanes(lanes)
g.upload_scene(scene)
for _ in range(4):
    g.render([cam], wave, outputs=outs)
g.synchronize()
g.set_async(True)
ts = []
s = torch.cuda.current_stream()
t00 = time.perf_counter()
for i in range(24):
    t0 = time.perf_counter()
    g.render([cam], wave, outputs=outs)
    ts.append(1e3 * (time.perf_counter() - t0))
g.join(s.cuda_stream)
torch.cuda.synchronize()
print(f"world {world} lanes {lanes}: total {1e3 * (time.perf_counter() - t00) / 24:.3f} ms/frame; host per call (ms):",
      " ".join(f"{t:.2f}" for t in ts))
g.frame_status()
