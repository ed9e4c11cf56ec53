"""Driver for ncu captures: warms up, then runs ONE C3 frame (or one training
iteration) inside an NVTX range "frame", so that

    ncu --set full --nvtx --nvtx-include "frame/" ... python tools/profile_frame.py [--train]

profiles exactly one unit of work.  Not a timing tool (numbers under ncu are
never bench values)."""
import argparse
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200.api import Context, Optimizer  # noqa: E402
from paper_2506_08350_b200.holotypes import PipelineOptions  # noqa: E402
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--train", action="store_true", help="one total_loss (with gradients) + optimizer step")
args = ap.parse_args()
c = CONFIGS[args.config]
wave, cam = c.wave(), c.cameras()[0]
ctx = Context(0)
ctx.upload_scene(synthetic_scene(c.n, wave, c.seed))
Lp, Cn, H, W = wave.num_planes, wave.channels(), wave.ny, wave.nx
if args.train:
    g = torch.Generator(device="cuda").manual_seed(0)
    targets = torch.rand((Lp, Cn, H, W), dtype=torch.float64, device="cuda", generator=g) * 0.1
    masks = (torch.rand((Lp, H, W), dtype=torch.float64, device="cuda", generator=g) > 0.7).double()
    opt, optim = PipelineOptions(), Optimizer(ctx)

    def unit():
        _, grads = ctx.total_loss(cam, wave, targets, masks, opt, n=c.n)
        optim.step(grads)
else:
    def unit():
        ctx.render(cam, wave, None, None, outputs=L.OUT_HOLOGRAM | L.OUT_INTENSITY)

for _ in range(2):
    unit()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("frame")
unit()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
