"""Time one training iteration on a BASELINE config: total_loss with gradients
(render + losses + pipeline backward + opacity term) and optimizer_step on the
resident scene, CUDA events on the context stream; plus holo_losses alone on the
same stacks.  Prints one JSON line."""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200.api import Context, Optimizer  # noqa: E402
from paper_2506_08350_b200.holotypes import OptimizerConfig, PipelineOptions  # noqa: E402
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
Lp, Cn, H, W = wave.num_planes, wave.channels(), wave.ny, wave.nx
gen = torch.Generator(device="cuda").manual_seed(0)
targets = torch.rand((Lp, Cn, H, W), dtype=torch.float64, device="cuda", generator=gen) * 0.1
masks = (torch.rand((Lp, H, W), dtype=torch.float64, device="cuda", generator=gen) > 0.7).double()
opt = PipelineOptions()
optim = Optimizer(ctx)
oc = OptimizerConfig()
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, n):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(n):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


holder = {}


def loss_step():
    b, g = ctx.total_loss(cam, wave, targets, masks, opt, n=c.n)
    holder["g"] = g
    holder["b"] = b


def train_step():
    loss_step()
    optim.step(holder["g"], oc)


ms_loss = timed(loss_step, args.steps)
ms_train = timed(train_step, args.steps)
I = torch.rand((Lp, Cn, H, W), dtype=torch.float64, device="cuda", generator=gen)
ms_losses = timed(lambda: ctx.losses(I, targets, masks, opt), args.steps)
ms_losses_nograd = timed(lambda: ctx.losses(I, targets, masks, opt, grad=False), args.steps)
print(json.dumps({"config": args.config, "total_loss_with_grads_ms": ms_loss, "train_step_ms": ms_train,
                  "optimizer_step_ms": ms_train - ms_loss, "losses_ms": ms_losses,
                  "losses_no_grad_ms": ms_losses_nograd, "loss": holder["b"].total,
                  "steps_taken": optim.counts()}))
