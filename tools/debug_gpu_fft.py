import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
import numpy as np
from paper_2506_08350_b200 import api
from paper_2506_08350_b200.holotypes import WaveConfig
from oracle.oracle import Oracle, rel_l2
ctx = api.Context(0)
rng = np.random.default_rng(1)
for n in [13, 17, 512, 1920, 1080, 8, 48, 128, 1000]:
    for shape in [(1, 1, n), (1, n, 1), (3, 1, n), (3, n, 1)]:
        x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        r = [rel_l2(ctx.fft2(x, False, p), np.fft.fft2(x)) for p in ("f64", "f32")]
        print(n, shape, ["%.1e" % v for v in r], flush=True)
ora = Oracle("restate")
for (w, h) in [(13, 17), (1920, 1080), (512, 384)]:
    cfg = WaveConfig(nx=w, ny=h, num_planes=2)
    u = rng.standard_normal((3, h, w)) + 1j * rng.standard_normal((3, h, w))
    print("prop", w, h, rel_l2(ctx.propagate(u, cfg, 1e-3, None, "f64"), ora.propagate(u, cfg, 1e-3)), flush=True)
