"""Multi-GPU partitioning of the render (one process per GPU, torch.distributed).

Plane sharding (BASELINE C3 at 1/2/4/8 GPUs): the hard plane assignment makes
every Gaussian belong to one depth plane (rasterizer.cpp:91-96), so rank g
rasterises planes [pb, pe) only, transforms them and forms its partial spectrum
S_g = sum_{l in g} H_{Z_l} FFT2(U_l).  Because forward_record is linear
(propagation.cpp:103-114), one all-reduce (sum) of S_g gives S, from which each
rank replays its own planes and rank 0 forms the hologram IFFT2(S)
(holo_render_begin / holo_render_end, include/holo_cuda.h).  Cost: C*H*W*8 bytes
per frame over NVLink (49.8 MB at C3).

View sharding (C4): frames are independent; each rank renders its slice of the
views with no per-frame collective.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def plane_ranges(num_planes: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous, balanced [pb, pe) plane ranges, one per rank (some may be empty)."""
    if world < 1:
        raise ValueError("world size must be positive")
    base, extra = divmod(num_planes, world)
    out, at = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((at, at + n))
        at += n
    return out


def hard_planes(scene):
    """Hard plane of every Gaussian with the device's strict '>' scan
    (preprocess.cu, ste_assign scene.cpp:132-152): ties and NaN logits keep the
    lower index, so every rank agrees with the kernel on who owns a Gaussian
    (np.argmax would return the first NaN instead)."""
    import numpy as np

    lg = np.asarray(scene.plane_logits, dtype=np.float64).reshape(scene.size(), scene.num_planes)
    best = np.zeros(lg.shape[0], dtype=np.int64)
    top = lg[:, 0].copy() if lg.shape[1] else np.zeros(0)
    for l in range(1, lg.shape[1]):
        take = lg[:, l] > top
        best[take] = l
        top[take] = lg[take, l]
    return best


def plane_subset(scene, pb: int, pe: int):
    """The Gaussians whose hard plane assignment (argmax of the plane logits, ties
    to the lowest index: ste_assign, scene.cpp:132-152) falls in [pb, pe), in
    their original order.  Under hard assignment a Gaussian contributes to its
    plane only, and the per-bucket order (depth, then index) is unchanged by an
    order-preserving subset, so a rank that uploads only this subset renders
    exactly the layers of the full scene for its planes -- with preprocessing
    and binning over ~N / world Gaussians instead of N."""
    import numpy as np

    from .holotypes import GaussianScene

    plane = hard_planes(scene)
    keep = (plane >= pb) & (plane < pe)
    sub = GaussianScene(num_planes=scene.num_planes)
    for k in ("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases", "plane_logits"):
        setattr(sub, k, np.ascontiguousarray(np.asarray(getattr(scene, k))[keep]))
    return sub


def view_ranges(num_views: int, world: int) -> List[Tuple[int, int]]:
    return plane_ranges(num_views, world)


class ShardedRenderer:
    """Plane-sharded frame: render_begin -> all_reduce(S) -> render_end.

    ``ctx`` is a paper_2506_08350_b200.api.Context on this rank's GPU with the scene
    uploaded; ``group`` a torch.distributed process group (NCCL on GPUs)."""

    def __init__(self, ctx, cfg, rank: int, world: int, group=None, outputs: int = None):
        import torch

        from . import _lib as L

        self.ctx, self.cfg, self.rank, self.world, self.group = ctx, cfg, rank, world, group
        self.pb, self.pe = plane_ranges(cfg.num_planes, world)[rank]
        self.outputs = outputs if outputs is not None else (L.OUT_INTENSITY | (L.OUT_HOLOGRAM if rank == 0 else 0))
        C, H, W = cfg.channels(), cfg.ny, cfg.nx
        self.spec = torch.empty((C, H, W, 2), dtype=torch.float32, device=f"cuda:{ctx.device}")

    def frame(self, cam, settings=None, prop=None) -> None:
        import torch.distributed as dist

        self.ctx.render_begin(cam, self.cfg, settings, prop, self.pb, self.pe, self.spec.data_ptr(), 0)
        if self.world > 1:
            dist.all_reduce(self.spec, group=self.group)
        self.ctx.render_end(self.cfg, prop, self.pb, self.pe, self.spec.data_ptr(), self.outputs)
