"""Plane sharding on CPU with world_size 2 over gloo.

Each rank takes its plane range (sharding.plane_ranges), forms the partial
spectrum S_g = sum_{l in g} H_{Z_l} FFT2(U_l) of the oracle's raster layers,
the ranks all-reduce S, and every rank checks that IFFT2(S) is the reference's
forward_record hologram and that its own planes replay as inverse_propagate
does -- the decomposition libholo_cuda's holo_render_begin / _end implement."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_08350_b200.sharding import plane_ranges, view_ranges


def test_plane_ranges_cover_and_balance():
    for L in range(1, 17):
        for world in range(1, 9):
            rs = plane_ranges(L, world)
            assert rs[0][0] == 0 and rs[-1][1] == L
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [e - b for b, e in rs]
            assert max(sizes) - min(sizes) <= 1
    assert view_ranges(64, 8) == [(8 * i, 8 * i + 8) for i in range(8)]


def test_plane_subsets_partition_the_scene_in_order():
    """sharding.plane_subset: the per-rank subsets partition the Gaussians by their
    hard plane (argmax of the logits, ties to the lowest plane) and keep the
    original relative order (which keeps every bucket's (depth, index) order)."""
    from paper_2506_08350_b200.holotypes import WaveConfig
    from paper_2506_08350_b200.scenes import synthetic_scene
    from paper_2506_08350_b200.sharding import plane_subset

    cfg = WaveConfig(nx=64, ny=64, num_planes=8)
    s = synthetic_scene(3000, cfg, 5)
    s.plane_logits[7, :] = 1.0  # an exact tie: goes to plane 0
    plane = np.argmax(s.plane_logits, axis=1)
    assert plane[7] == 0
    for world in (1, 2, 4, 8):
        parts = [plane_subset(s, pb, pe) for pb, pe in plane_ranges(8, world)]
        assert sum(p.size() for p in parts) == s.size()
        for (pb, pe), p in zip(plane_ranges(8, world), parts):
            idx = np.nonzero((plane >= pb) & (plane < pe))[0]
            assert np.array_equal(p.positions, s.positions[idx])  # same rows, same order
            assert np.array_equal(p.plane_logits, s.plane_logits[idx])


def test_hard_planes_follow_the_kernels_strict_scan():
    """NaN logits never win the device's strict '>' scan (preprocess.cu), so a
    NaN in front keeps plane 0 and a NaN later is skipped; ties keep the lower
    plane.  np.argmax would send the first row to plane 1."""
    from paper_2506_08350_b200.holotypes import GaussianScene
    from paper_2506_08350_b200.sharding import hard_planes

    s = GaussianScene(num_planes=4)
    s.resize(5)
    s.plane_logits = np.array([[0.0, np.nan, 1.0, 0.5],
                               [np.nan, 2.0, 3.0, 1.0],
                               [1.0, 1.0, 1.0, 1.0],
                               [0.0, 0.0, 0.0, 5.0],
                               [np.nan, np.nan, np.nan, np.nan]])
    assert hard_planes(s).tolist() == [2, 0, 0, 3, 0]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle.oracle import Oracle
    from paper_2506_08350_b200.holotypes import WaveConfig
    from paper_2506_08350_b200.scenes import front_camera, synthetic_scene

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ora = Oracle("restate")
    cfg = WaveConfig(nx=48, ny=40, num_planes=4)
    scene = synthetic_scene(400, cfg, 9)
    cam = front_camera(cfg)
    z = ora.plane_positions(cfg)
    layers = ora.raster_forward(scene, cam, cfg).layers  # [L, 3, H, W]
    pb, pe = plane_ranges(cfg.num_planes, world)[rank]
    S = np.zeros((3, cfg.ny, cfg.nx), dtype=np.complex128)
    for l in range(pb, pe):
        S += ora.transfer_function(cfg, z[l]) * np.fft.fft2(layers[l])
    t = torch.from_numpy(np.ascontiguousarray(S).view(np.float64).copy())
    dist.all_reduce(t)
    S = t.numpy().view(np.complex128).reshape(3, cfg.ny, cfg.nx)
    holo = np.fft.ifft2(S)
    ref_holo = ora.forward_record(layers, cfg)
    ok_holo = float(np.abs(holo - ref_holo).max() / np.abs(ref_holo).max())
    ref_rep = ora.inverse_propagate(ref_holo, cfg)
    ok_rep = 0.0
    for l in range(pb, pe):
        rep = np.fft.ifft2(np.conj(ora.transfer_function(cfg, z[l])) * S)
        ok_rep = max(ok_rep, float(np.abs(rep - ref_rep[l]).max() / np.abs(ref_rep[l]).max()))
    out[rank] = (ok_holo, ok_rep, pe - pb)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_plane_sharding():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert sum(out[r][2] for r in range(2)) == 4
    for r in range(2):
        assert out[r][0] < 1e-12 and out[r][1] < 1e-12


def test_mesh_layout_library_equals_python_statement():
    """holo_mesh_layout (group.cu, pure host arithmetic through the C-ABI) against
    sharding.mesh for every small mesh: plane and view ranges, plane rank, view
    group and hologram channel owners."""
    from paper_2506_08350_b200.api import mesh_layout
    from paper_2506_08350_b200.sharding import mesh

    for world in range(1, 9):
        for ps in [d for d in range(1, world + 1) if world % d == 0]:
            for L in (1, 3, 6, 8, 16):
                for V in (1, 5, 64):
                    for C in (1, 3):
                        for r in range(world):
                            m = mesh_layout(world, r, ps, L, V, C)
                            want = mesh(world, r, ps, L, V, C)
                            got = {k: getattr(m, k) for k, _ in m._fields_}
                            assert got == want, (world, ps, L, V, C, r)
    with pytest.raises(Exception):
        mesh_layout(6, 0, 4, 8)  # plane split must divide the world


def _mesh_worker(rank, world, ps, port, out):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2506_08350_b200.api import mesh_layout
    from paper_2506_08350_b200.sharding import torch_plane_group

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pg = torch_plane_group(ps)
    m = mesh_layout(world, rank, ps, 16, 64, 3)
    # the plane group sums exactly the ranks sharing this rank's view group, and
    # their plane ranges tile [0, 16)
    t = torch.tensor([float(rank), float(m.plane_end - m.plane_begin), float(m.view_group)])
    dist.all_reduce(t, group=pg)
    members = list(range(m.view_group * ps, (m.view_group + 1) * ps))
    out[rank] = (t[0].item() == sum(members), t[1].item() == 16, t[2].item() == m.view_group * ps,
                 m.view_end - m.view_begin)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,ps", [(2, 2), (2, 1), (4, 2)])
def test_gloo_mesh_plane_groups(world, ps):
    """The planes x views mesh of the C-ABI group under torch.distributed (gloo):
    plane groups from sharding.torch_plane_group agree with holo_mesh_layout."""
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_mesh_worker, args=(r, world, ps, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    for r in range(world):
        assert out[r][:3] == (True, True, True)
    assert sum(out[r][3] for r in range(0, world, ps)) == 64
