"""Host vs device time per frame: Context.render against Group.render (world 1)
on C3 -- is the group path's enqueue host-bound?"""
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
s = torch.cuda.current_stream()


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    return (t1 - t0) * 1e3 / n, e0.elapsed_time(e1) / n


ctx = Context(0)
ctx.upload_scene(scene)
ctx.render(cam, wave, outputs=outs)
ctx.set_async(True)
print("ctx.render async: host %.3f ms, device %.3f ms" % timeit(lambda: ctx.render(cam, wave, outputs=outs)))
ctx.frame_status()
ctx.close()
for mode in ("nccl", "callback"):
    ctx = Context(0)
    g = Group(ctx) if mode == "nccl" else Group(ctx, 1, 0, 1, allreduce=lambda *a: 0)
    g.upload_scene(scene)
    g.render([cam], wave, outputs=outs)
    g.synchronize()
    print(f"group[{mode}] sync: host %.3f ms, device %.3f ms" % timeit(lambda: g.render([cam], wave, outputs=outs)))
    g.set_async(True)
    print(f"group[{mode}] async: host %.3f ms, device %.3f ms" % timeit(lambda: g.render([cam], wave, outputs=outs)))
    g.frame_status()
    for flags in (L.GROUP_SHARDED_PATH,):
        print(f"group[{mode}] sharded-path async: host %.3f ms, device %.3f ms" % timeit(
            lambda: g.render([cam], wave, outputs=outs, flags=flags)))
    g.frame_status()
    g.close()
    ctx.close()
