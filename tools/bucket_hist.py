"""Histogram of bucket sizes (entries per (plane, tile) work list) of one frame:
the input distribution the per-bucket sorts and the compositing kernel see.

  python tools/bucket_hist.py [--config C3]"""
import argparse
import json
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200.api import Context  # noqa: E402
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
args = ap.parse_args()
c = CONFIGS[args.config]
wave, cam = c.wave(), c.cameras()[0]
ctx = Context(0)
ctx.upload_scene(synthetic_scene(c.n, wave, c.seed))
ctx.render(cam, wave, outputs=L.OUT_HOLOGRAM | L.OUT_LISTS)
tiles = ((wave.nx + 15) // 16) * ((wave.ny + 15) // 16)
B = tiles * wave.num_planes
bs = ctx.download(L.BUF_BUCKET_START, np.uint32, (B + 1,)).astype(np.int64)
n = np.diff(bs)
edges = [0, 1, 2, 8, 16, 32, 64, 128, 256, 1024, 1 << 30]
hist = {f"{lo}-{hi - 1}": [int(((n >= lo) & (n < hi)).sum()), int(n[(n >= lo) & (n < hi)].sum())]
        for lo, hi in zip(edges[:-1], edges[1:])}
print(json.dumps({"config": args.config, "buckets": int(B), "entries": int(n.sum()), "mean": float(n.mean()),
                  "buckets_entries_by_size": hist}))
ctx.close()
