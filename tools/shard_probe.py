"""One rank's share of a sharded frame, timed on one GPU without its collective:
the product path (holo_group_render through a callback transport whose "sum" is a
no-op), so the rank runs exactly its kernels of an N-GPU job -- device-side plane
subset, per-channel partial spectra, per-channel replays, its hologram channels --
and the timing shows how the per-rank compute shrinks with N.  The spectrum sums
(C pieces of P complex64, overlapped with the row pass in the real job) come on
top at N > 1.

  python tools/shard_probe.py [--config C3] [--lanes 1]
prints {"rank_frame_ms": {N: ms}} for rank 0 (the most planes and hologram
channel 0) and each rank's share at N = 8."""
import argparse
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200.api import Context, Group  # noqa: E402
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--lanes", type=int, default=1)
ap.add_argument("--frames", type=int, default=20)
args = ap.parse_args()
c = CONFIGS[args.config]
wave, cam = c.wave(), c.cameras()[0]
scene = synthetic_scene(c.n, wave, c.seed)
outs = L.OUT_INTENSITY | L.OUT_HOLOGRAM


def rank_ms(world, rank):
    ctx = Context(0)
    g = Group(ctx, world, rank, world, allreduce=lambda *a: 0)  # planes only; the sum skipped
    if args.lanes > 1:
        g.set_lanes(args.lanes)
    g.upload_scene(scene)
    flags = 0  # N = 1: the unsharded frame
    for _ in range(3):
        g.render([cam], wave, outputs=outs, flags=flags)
    g.synchronize()
    g.set_async(True)
    for _ in range(2 * max(1, args.lanes)):  # every lane's first asynchronous frame grows its buffers
        g.render([cam], wave, outputs=outs, flags=flags)
    g.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(args.frames):
        g.render([cam], wave, outputs=outs, flags=flags)
    g.join(s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    g.frame_status()
    g.close()
    ctx.close()
    return e0.elapsed_time(e1) / args.frames


res = {N: rank_ms(N, 0) for N in (1, 2, 4, 8)}
per_rank8 = [rank_ms(8, r) for r in range(8)]
print(json.dumps({"config": args.config, "rank_frame_ms": res, "n8_rank_ms": per_rank8}))
