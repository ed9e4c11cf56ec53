"""Multi-GPU partitioning of the render (one process per GPU, torch.distributed).

Plane sharding (BASELINE C3 at 1/2/4/8 GPUs): the hard plane assignment makes
every Gaussian belong to one depth plane (rasterizer.cpp:91-96), so rank g
rasterises planes [pb, pe) only, transforms them and forms its partial spectrum
S_g = sum_{l in g} H_{Z_l} FFT2(U_l) channel by channel.  Because forward_record
is linear (propagation.cpp:103-114), the sum of S_g over the plane group gives S;
channel c is summed while the row pass of channel c + 1 runs, then each rank
replays its own planes and forms the hologram channels c with c mod plane_split
== its plane rank (holo_group_render, include/holo_cuda.h; the lower-level
holo_render_begin / _end split one frame around a caller's collective).  Cost:
C*H*W*8 bytes per frame over NVLink (49.8 MB at C3).

View sharding (C4): frames are independent; each rank renders its slice of the
views with no per-frame collective.  Planes x views (C5): world = view groups x
plane split, the sum inside each plane group.
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


def mesh(world: int, rank: int, plane_split: int, num_planes: int, num_views: int = 1, channels: int = 3) -> dict:
    """Python statement of holo_mesh_layout (group.cu): world = view_groups x
    plane_split; rank r is plane rank r % plane_split of view group r // plane_split;
    it renders its plane group's share of the planes and its view group's share of
    the views, and forms hologram channel c when c % plane_split is its plane rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank outside [0, world)")
    if plane_split < 1 or world % plane_split:
        raise ValueError("plane_split must divide the world size")
    vg = world // plane_split
    pr, v = rank % plane_split, rank // plane_split
    pb, pe = plane_ranges(num_planes, plane_split)[pr]
    vb, ve = view_ranges(num_views, vg)[v]
    holo = sum(1 << c for c in range(channels) if c % plane_split == pr)
    return {"world": world, "rank": rank, "plane_split": plane_split, "view_groups": vg, "plane_rank": pr,
            "view_group": v, "plane_begin": pb, "plane_end": pe, "view_begin": vb, "view_end": ve,
            "holo_channels": holo}


def plane_groups(world: int, plane_split: int):
    """Rank lists of the plane groups (the all-reduce groups of the spectrum)."""
    return [list(range(g * plane_split, (g + 1) * plane_split)) for g in range(world // plane_split)]


def torch_plane_group(plane_split: int):
    """This rank's torch.distributed plane group (every rank creates all of them,
    as new_group requires); None for plane groups of one."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    mine = None
    for ranks in plane_groups(world, plane_split):
        pg = dist.new_group(ranks)
        if rank in ranks:
            mine = pg
    return mine


class ShardedRenderer:
    """A frame split over the ranks of a torch.distributed job through the C-ABI
    group (holo_group_*): planes (plane_split = world), views (plane_split = 1) or
    planes x views.  transport "nccl" builds the library's own NCCL communicators
    (unique id broadcast from rank 0); "gloo" sums the spectrum through torch's
    gloo plane group (every rank may share one GPU -- the tests)."""

    def __init__(self, ctx, cfg, plane_split: int = None, transport: str = "nccl", lanes: int = 1):
        import torch.distributed as dist

        from .api import Group, gloo_allreduce

        self.ctx, self.cfg = ctx, cfg
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        self.plane_split = self.world if plane_split is None else plane_split
        if transport == "nccl":
            self.group = Group.from_torch(ctx, self.plane_split)
        else:
            pg = torch_plane_group(self.plane_split)
            self.group = Group(ctx, self.world, self.rank, self.plane_split, allreduce=gloo_allreduce(pg))
        if lanes > 1:
            self.group.set_lanes(lanes)

    def upload_scene(self, scene) -> None:
        self.group.upload_scene(scene)

    def mesh(self, num_views: int = 1):
        return self.group.mesh(self.cfg.num_planes, num_views, self.cfg.channels())

    def frame(self, cams, settings=None, prop=None, outputs: int = None, flags: int = 0, view_outputs=None):
        from . import _lib as L

        cams = cams if isinstance(cams, (list, tuple)) else [cams]
        outs = L.OUT_HOLOGRAM | L.OUT_INTENSITY if outputs is None else outputs
        return self.group.render(cams, self.cfg, settings, prop, outs, flags, view_outputs)

    def close(self):
        self.group.close()
