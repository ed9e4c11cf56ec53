"""Stage times (CUDA events) of rank 0's share of a plane-sharded C3 frame at N GPUs,
timed on one GPU through holo_group_render with a no-op sum."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200.api import Context, Group  # noqa: E402
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene  # noqa: E402

c = CONFIGS["C3"]
wave, cam = c.wave(), c.cameras()[0]
scene = synthetic_scene(c.n, wave, c.seed)
outs = L.OUT_INTENSITY | L.OUT_HOLOGRAM
for N in (1, 8):
    ctx = Context(0)
    g = Group(ctx, N, 0, N, allreduce=lambda *a: 0)
    g.upload_scene(scene)
    for _ in range(4):
        g.render([cam], wave, outputs=outs)
    g.synchronize()
    ctx.reset_timing()
    ctx.enable_timing(True)
    for _ in range(10):
        g.render([cam], wave, outputs=outs)
    g.synchronize()
    st = ctx.stage_times()
    print(json.dumps({"N": N, "stages_ms_per_frame": {k: round(v[0] / 10, 4) for k, v in st.items()},
                      "launches_per_frame": {k: v[1] / 10 for k, v in st.items()}}))
    g.close()
    ctx.close()
