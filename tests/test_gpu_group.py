"""GPU tests of the multi-GPU group renderer (holo_group_*, group.cu): plane
sharding, view sharding and the planes x views mesh, against single-GPU frames
(holo_render, itself checked against the oracle in test_gpu_render.py).

By the linearity of forward_record (propagation.cpp:103-114) a plane-sharded
frame equals the single-GPU frame up to the fp32 summation order of the
spectrum.  One box has one GPU, so:
  * world 1 runs the NCCL transport for real (a one-rank communicator) with
    HOLO_GROUP_SHARDED_PATH forcing the per-channel sharded pipeline;
  * worlds 2 and 4 run one process per rank, all on cuda:0, with the library's
    callback transport summing through torch's gloo plane groups (NCCL refuses
    two ranks on one device).  Every rank drives the product path
    (holo_group_render: device-side scene subset, per-channel spectrum, sum,
    replay, hologram channel owners) and compares its share with the full frame.
"""
import os
import socket

import numpy as np
import pytest

from conftest import rel_l2
from paper_2506_08350_b200 import _lib as L
from paper_2506_08350_b200 import api
from paper_2506_08350_b200.holotypes import WaveConfig
from paper_2506_08350_b200.scenes import front_camera, synthetic_scene

pytestmark = pytest.mark.gpu
RGB = (639e-9, 532e-9, 473e-9)


def _views(cfg, n):
    return [front_camera(cfg, yaw=-0.1 + 0.2 * k / max(1, n - 1)) for k in range(n)]


def _full(ctx, cam, cfg):
    ctx.render(cam, cfg, outputs=L.OUT_HOLOGRAM | L.OUT_INTENSITY)
    C, H, W = cfg.channels(), cfg.ny, cfg.nx
    return (ctx.download(L.BUF_HOLOGRAM, np.complex64, (C, H, W)),
            ctx.download(L.BUF_INTENSITY, np.float32, (cfg.num_planes, C, H, W)))


@pytest.mark.parametrize("W,H,L_", [(256, 192, 4), (96, 80, 3)])  # static plans; runtime-planned sizes
def test_world1_nccl_sharded_path_equals_render(W, H, L_):
    import torch

    cfg = WaveConfig(nx=W, ny=H, wavelengths=RGB, num_planes=L_)
    scene = synthetic_scene(20000, cfg, 61)
    cam = front_camera(cfg)
    ctx = api.Context(0)
    g = api.Group(ctx)  # world 1: NCCL communicator of one rank
    g.upload_scene(scene)
    holo_ref, int_ref = _full(ctx, cam, cfg)
    C = cfg.channels()
    hh = torch.empty((C, H, W), dtype=torch.complex64, device="cuda:0")
    ii = torch.empty((L_, C, H, W), dtype=torch.float32, device="cuda:0")
    infos = g.render([cam], cfg, outputs=L.OUT_HOLOGRAM | L.OUT_INTENSITY, flags=L.GROUP_SHARDED_PATH,
                     view_outputs={0: (hh, None, ii)})
    g.synchronize()
    assert infos[0].num_entries > 0
    assert rel_l2(hh.cpu().numpy(), holo_ref) < 1e-6
    assert rel_l2(ii.cpu().numpy(), int_ref) < 1e-6
    g.close()
    ctx.close()


def test_world1_views_with_lanes_equal_single_frames():
    """A 6-view batch on one rank with two lanes (frames in flight on two streams,
    the scene replicated on the device): every view equals holo_render of it."""
    import torch

    cfg = WaveConfig(nx=256, ny=256, wavelengths=RGB, num_planes=3)
    scene = synthetic_scene(30000, cfg, 62)
    cams = _views(cfg, 6)
    ctx = api.Context(0)
    g = api.Group(ctx, plane_split=1)
    g.set_lanes(2)
    g.upload_scene(scene)
    C = cfg.channels()
    outs = {v: (torch.empty((C, 256, 256), dtype=torch.complex64, device="cuda:0"), None,
                torch.empty((3, C, 256, 256), dtype=torch.float32, device="cuda:0")) for v in range(6)}
    infos = g.render(cams, cfg, view_outputs=outs)
    g.synchronize()
    ref_ctx = api.Context(0)
    ref_ctx.upload_scene(scene)
    for v, cam in enumerate(cams):
        holo, ints = _full(ref_ctx, cam, cfg)
        assert infos[v].num_entries == ref_ctx.info.num_entries
        assert np.array_equal(outs[v][0].cpu().numpy(), holo)
        assert np.array_equal(outs[v][2].cpu().numpy(), ints)
    g.close()
    ctx.close()
    ref_ctx.close()


def test_group_rejects_bad_meshes():
    ctx = api.Context(0)
    with pytest.raises(L.HoloError):
        api.Group(ctx, world=4, rank=0, plane_split=3, allreduce=lambda *a: 0)
    with pytest.raises(L.HoloError):
        api.Group(ctx, world=2, rank=2, allreduce=lambda *a: 0)
    g = api.Group(ctx)
    cfg = WaveConfig(nx=64, ny=64, wavelengths=RGB, num_planes=2)
    g.upload_scene(synthetic_scene(100, cfg, 1))
    from paper_2506_08350_b200.holotypes import PropagationOptions

    with pytest.raises(L.HoloError):  # the spectrum shortcut needs pad2x off
        g.render([front_camera(cfg)], cfg, prop=PropagationOptions(pad2x=True), flags=L.GROUP_SHARDED_PATH)
    g.close()
    ctx.close()


# ---------------------------------------------------------------- worlds 2 and 4 on one GPU (gloo transport)

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_worker(rank, world, ps, L_, V, gather, port, out):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch
    import torch.distributed as dist

    from paper_2506_08350_b200.sharding import ShardedRenderer

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        cfg = WaveConfig(nx=128, ny=128, wavelengths=RGB, num_planes=L_)
        scene = synthetic_scene(15000, cfg, 70)
        cams = _views(cfg, V)
        ctx = api.Context(0)
        sr = ShardedRenderer(ctx, cfg, plane_split=ps, transport="gloo")
        sr.upload_scene(scene)
        m = sr.mesh(V)
        C, np_ = cfg.channels(), m.plane_end - m.plane_begin
        outs = {v: (torch.zeros((C, 128, 128), dtype=torch.complex64, device="cuda:0"), None,
                    torch.zeros((max(np_, 1), C, 128, 128), dtype=torch.float32, device="cuda:0"))
                for v in range(m.view_begin, m.view_end)}
        flags = L.GROUP_GATHER_HOLOGRAM if gather else 0
        sr.frame(cams, flags=flags, view_outputs=outs)
        sr.group.synchronize()
        ref_ctx = api.Context(0)
        ref_ctx.upload_scene(scene)
        errs = []
        for v in range(m.view_begin, m.view_end):
            holo, ints = _full(ref_ctx, cams[v], cfg)
            gh = outs[v][0].cpu().numpy()
            chans = range(C) if gather else [c for c in range(C) if (m.holo_channels >> c) & 1]
            for c in chans:
                errs.append(rel_l2(gh[c], holo[c]))
            if np_:
                errs.append(rel_l2(outs[v][2].cpu().numpy()[:np_], ints[m.plane_begin:m.plane_end]))
        out[rank] = (max(errs) if errs else 0.0, np_, m.view_end - m.view_begin, len(errs))
        sr.close()
        ctx.close()
        ref_ctx.close()
    except Exception as e:  # noqa: BLE001
        out[rank] = (repr(e), 0, 0, 0)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,ps,L_,V,gather", [
    (2, 2, 4, 1, False),   # planes: 2 + 2, hologram channels 0, 2 | 1
    (2, 2, 3, 2, True),    # uneven planes (2 + 1), two views, gathered hologram
    (2, 1, 4, 3, False),   # views only: 2 + 1 views
    (4, 2, 4, 4, False),   # planes x views: 2 view groups x 2 plane ranks
    (4, 4, 3, 1, True),    # more ranks than planes: rank 3 renders no plane
])
def test_group_ranks_on_one_gpu_equal_single_gpu_frames(world, ps, L_, V, gather):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, ps, L_, V, gather, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    for r in range(world):
        assert not isinstance(out[r][0], str), out[r][0]
        assert out[r][0] < 1e-5, (r, out[r])
    # planes of a plane group tile [0, L); views of the view groups tile [0, V)
    assert sum(out[r][1] for r in range(ps)) == L_
    assert sum(out[r][2] for r in range(0, world, ps)) == V
