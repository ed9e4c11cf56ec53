"""Time the gradient branch (holo_pipeline_backward) on a BASELINE config: one
render with the outputs the backward needs, then the backward alone, CUDA events
on the context stream.  Prints one JSON line."""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200.api import Context  # noqa: E402
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
c = CONFIGS[args.config]
wave, cam = c.wave(), c.cameras()[0]
scene = synthetic_scene(c.n, wave, c.seed)
ctx = Context(0)
ctx.upload_scene(scene)
outs = L.OUT_HOLOGRAM | L.OUT_INTENSITY | L.OUT_REPLAYED | L.OUT_AUX
Lp, Cn, H, W = wave.num_planes, wave.channels(), wave.ny, wave.nx
gi = torch.randn((Lp, Cn, H, W), dtype=torch.float32, device="cuda")
ctx.render(cam, wave, None, None, outputs=outs)
ctx.enable_timing(False)
for _ in range(2):
    ctx.pipeline_backward(cam, wave, None, None, gi, c.n)
torch.cuda.synchronize()
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(args.steps):
    ctx.pipeline_backward(cam, wave, None, None, gi, c.n)
e1.record(s)
torch.cuda.synchronize()
ms_bwd = e0.elapsed_time(e1) / args.steps
e0.record(s)
for _ in range(args.steps):
    ctx.render(cam, wave, None, None, outputs=outs)
e1.record(s)
torch.cuda.synchronize()
ms_fwd = e0.elapsed_time(e1) / args.steps
print(json.dumps({"config": args.config, "forward_ms (render with replayed + aux outputs)": ms_fwd,
                  "backward_ms (pipeline_backward)": ms_bwd, "entries": int(ctx.info.num_entries)}))
