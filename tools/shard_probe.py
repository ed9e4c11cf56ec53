"""One rank's share of a plane-sharded C3 frame, timed on one GPU (no collective):
holo_render_begin for planes [0, L/N) and holo_render_end with the hologram and
those planes' intensities, the rank holding only its planes' Gaussians
(sharding.plane_subset, as bench.py's sharded runs do).  Estimates how the per-rank compute shrinks with N; the
all-reduce of the 49.8 MB spectrum comes on top at N > 1."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200.api import Context  # noqa: E402
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene  # noqa: E402

c = CONFIGS["C3"]
wave, cam = c.wave(), c.cameras()[0]
scene = synthetic_scene(c.n, wave, c.seed)
ctx = Context(0)
ctx.upload_scene(scene)
Cn, H, W, Lp = wave.channels(), wave.ny, wave.nx, wave.num_planes
spec = torch.zeros((Cn, H, W, 2), dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
res = {}
from paper_2506_08350_b200.sharding import plane_subset  # noqa: E402

for N in (1, 2, 4, 8):
    pe = Lp // N
    outs = L.OUT_INTENSITY | L.OUT_HOLOGRAM
    ctx.upload_scene(plane_subset(scene, 0, pe) if N > 1 else scene)

    def frame():
        ctx.render_begin(cam, wave, None, None, 0, pe, spec.data_ptr(), 0)
        ctx.render_end(wave, None, 0, pe, spec.data_ptr(), outs)

    for _ in range(3):
        frame()
    ctx.set_async(True)
    for _ in range(2):
        frame()
    ctx.frame_status()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20):
        frame()
    e1.record(s)
    torch.cuda.synchronize()
    ctx.frame_status()
    ctx.set_async(False)
    res[N] = e0.elapsed_time(e1) / 20
print(json.dumps({"rank_frame_ms": res}))

# stage split of the N = 8 share
pe = Lp // 8
ctx.reset_timing()
ctx.enable_timing(True)
for _ in range(10):
    ctx.render_begin(cam, wave, None, None, 0, pe, spec.data_ptr(), 0)
    ctx.render_end(wave, None, 0, pe, spec.data_ptr(), L.OUT_INTENSITY | L.OUT_HOLOGRAM)
st = ctx.stage_times()
print(json.dumps({k: round(v[0] / max(v[1], 1), 4) for k, v in st.items()}))
