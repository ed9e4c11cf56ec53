"""Time convert_phase_only on the GPU for a hologram of a BASELINE config (the
config's rendered hologram, its optics and plane stack, pad2x as the reference's
default), per iteration; optionally time the reference build on a small sample.
Prints one JSON line."""
import argparse
import json
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200.api import Context  # noqa: E402
from paper_2506_08350_b200.holotypes import PhaseOnlyOptions, PropagationOptions  # noqa: E402
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--no-pad", action="store_true")
args = ap.parse_args()
c = CONFIGS[args.config]
wave, cam = c.wave(), c.cameras()[0]
ctx = Context(0)
ctx.upload_scene(synthetic_scene(c.n, wave, c.seed))
ctx.render(cam, wave, None, None, outputs=L.OUT_HOLOGRAM)
Cn, H, W = wave.channels(), wave.ny, wave.nx
P = ctx.tensor(L.BUF_HOLOGRAM, "c8", (Cn, H, W)).to(torch.complex128).clone()
opt = PhaseOnlyOptions(prop=PropagationOptions(pad2x=not args.no_pad))
ctx.convert_phase_only(P, wave, 1, 0.02, opt)  # warm-up: buffers, plans
torch.cuda.synchronize()
t0 = time.perf_counter()
_, trace = ctx.convert_phase_only(P, wave, args.iters, 0.02, opt)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(json.dumps({"config": args.config, "grid": [W, H], "planes": wave.num_planes, "channels": Cn,
                  "pad2x": not args.no_pad, "iters": args.iters, "s_total": dt,
                  "ms_per_iter": 1e3 * dt / (args.iters + 1), "trace_first": trace[0], "trace_best": min(trace)}))
