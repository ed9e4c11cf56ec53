"""GPU parity of the forward render (holo_render = pipeline_forward /
raster_forward, pipeline.cpp:20-29, rasterizer.cpp:139-263) against the C
restatement of the reference, on identical synthetic scenes.

Bars (north star): complex fields rel-L2 <= 1e-4 (fp32 vs f64), intensity PSNR
within 0.01 dB, per-tile work lists (entries, bucket_start) bit-exact, f64
projections of centres and depths bit-exact."""
import math

import numpy as np
import pytest

from conftest import desk_config, front_camera, mild_posed_camera, overlapping_scene, random_scene, rel_l2, \
    single_scene
from oracle.oracle import psnr
from paper_2506_08350_b200 import _lib as L
from paper_2506_08350_b200 import api
from paper_2506_08350_b200._lib import HoloError
from paper_2506_08350_b200.holotypes import PipelineOptions, PropagationOptions, RenderSettings, WaveConfig
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene
from paper_2506_08350_b200.scenes import front_camera as wide_camera

pytestmark = pytest.mark.gpu
RGB = (639e-9, 532e-9, 473e-9)


def check_pipeline(ctx, oracle, scene, cam, cfg, st=None, prop=None, tol=1e-4, lists=True):
    st = st or RenderSettings()
    prop = prop or PropagationOptions()
    g = api.pipeline_forward(scene, cam, cfg, PipelineOptions(raster=st, prop=prop), ctx=ctx)
    r = oracle.pipeline_forward(scene, cam, cfg, st, prop)
    C = cfg.channels()
    errs = {"layers": rel_l2(np.stack(g.raster.layers), r.raster.layers[:, :C]),
            "hologram": rel_l2(g.hologram, r.hologram),
            "replayed": rel_l2(np.stack(g.replayed), r.replayed),
            "intensity": rel_l2(np.stack(g.intensities), r.intensities)}
    for k, v in errs.items():
        assert v <= tol, (k, v)
    ints = np.stack(g.intensities)
    for l in range(cfg.num_planes):
        t = 0.9025 * r.intensities[l]  # target: the same scene with amplitudes x 0.95
        assert abs(psnr(ints[l], t) - psnr(r.intensities[l], t)) <= 0.01
    if lists:
        assert np.array_equal(g.raster.bucket_start, r.raster.bucket_start)
        assert np.array_equal(g.raster.entries["gidx"], r.raster.entry_gidx)
        assert np.array_equal(g.raster.entries["bucket"], r.raster.entry_bucket)
        assert np.array_equal(g.raster.entries["depth"], r.raster.entry_depth)
        for k in ("valid", "plane", "mu_x", "mu_y", "zc", "xc", "yc"):
            assert np.array_equal(g.raster.projected[k], r.raster.projected[k]), k
        for k in ("inv00", "inv01", "inv11", "radius", "alpha_sig"):
            # CUDA's f64 exp/log may differ from glibc's by an ulp; inv01 carries
            # cancellation, so scale the bound by the conic's magnitude
            ref = r.raster.projected[k]
            scale = np.abs(ref).max() if ref.size else 0.0
            assert np.allclose(g.raster.projected[k], ref, rtol=1e-12, atol=1e-12 * scale), k
        assert np.array_equal(g.raster.touched, r.raster.touched)
        assert np.array_equal(g.raster.rho, r.raster.rho)
    # Contribution counts and final transmittance: an fp32 alpha within an ulp of
    # alpha_floor (or of term_eps for T) can flip one accept decision, which moves T
    # of that pixel by a factor (1 - 1/255).  Such pixels must stay rare.  With no
    # floor (alpha_floor <= 0) the reference also counts contributions below fp32's
    # normal range, so only the fields are compared.
    if st.alpha_floor > 0:
        mism = np.count_nonzero(g.raster.n_contrib != r.raster.n_contrib)
        assert mism <= max(3, 2e-4 * g.raster.n_contrib.size), mism
        dT = np.abs(g.raster.t_final - r.raster.t_final)
        assert np.count_nonzero(dT > 1e-4) <= max(3, 2e-4 * dT.size)
        assert dT.max() < 0.01
    return g, r, errs


@pytest.mark.parametrize("n,W,H,L,wl,seed", [
    (300, 64, 48, 3, RGB, 1),
    (3000, 256, 256, 3, (515e-9,), 2),        # C1-like, single wavelength adapter
    (20000, 512, 384, 4, (638e-9, 520e-9, 450e-9), 3),
    (800, 96, 80, 2, RGB, 4),                 # generic (runtime-planned) FFT sizes
    (500, 30, 42, 5, RGB, 5),                 # ragged tiles, odd grid
    (0, 64, 64, 2, RGB, 6),                   # empty scene
    (1, 64, 64, 1, RGB, 7),                   # one Gaussian, one plane
])
def test_pipeline_parity(gpu_ctx, oracle, n, W, H, L, wl, seed):
    cfg = WaveConfig(nx=W, ny=H, wavelengths=wl, num_planes=L)
    check_pipeline(gpu_ctx, oracle, synthetic_scene(n, cfg, seed), wide_camera(cfg), cfg)


@pytest.mark.parametrize("tile", [8, 16, 32])
def test_tile_sizes(gpu_ctx, oracle, tile):
    cfg = WaveConfig(nx=96, ny=64, wavelengths=RGB, num_planes=3)
    check_pipeline(gpu_ctx, oracle, synthetic_scene(1500, cfg, 10 + tile), wide_camera(cfg), cfg,
                   RenderSettings(tile=tile))


def test_soft_assignment(gpu_ctx, oracle):
    cfg = WaveConfig(nx=64, ny=64, wavelengths=RGB, num_planes=3)
    st = RenderSettings(soft_assignment=True, soft_tau=1.0)
    check_pipeline(gpu_ctx, oracle, synthetic_scene(400, cfg, 21), wide_camera(cfg), cfg, st)


def test_gradcheck_settings(gpu_ctx, oracle):
    # helpers.hpp:105-111: no floor, no termination, wide cutoff
    cfg = WaveConfig(nx=48, ny=48, wavelengths=RGB, num_planes=2)
    st = RenderSettings(alpha_floor=0.0, term_eps=0.0, radius_form_cap=80.0)
    check_pipeline(gpu_ctx, oracle, random_scene(40, cfg, 22), front_camera(cfg), cfg, st)


def test_posed_camera_and_reference_helpers(gpu_ctx, oracle):
    cfg = WaveConfig(nx=48, ny=48, num_planes=2)
    check_pipeline(gpu_ctx, oracle, random_scene(60, cfg, 23), mild_posed_camera(cfg), cfg)
    check_pipeline(gpu_ctx, oracle, overlapping_scene(40, cfg, 24), front_camera(cfg), cfg)


@pytest.mark.parametrize("local", [False, True])
def test_evanescent_band_pipeline(gpu_ctx, oracle, local):
    # pitch 0.3 um: the grid's corner frequencies exceed 1/lambda, so H = 0 there
    # (propagation.cpp:41-44); with local band limits on, the per-plane limits too
    cfg = WaveConfig(nx=64, ny=48, pitch=0.3e-6, wavelengths=RGB, num_planes=3)
    check_pipeline(gpu_ctx, oracle, synthetic_scene(500, cfg, 26), wide_camera(cfg), cfg,
                   prop=PropagationOptions(local_band_limit=local))


def test_pad2x_pipeline(gpu_ctx, oracle):
    cfg = WaveConfig(nx=48, ny=32, wavelengths=RGB, num_planes=2)
    check_pipeline(gpu_ctx, oracle, synthetic_scene(200, cfg, 25), wide_camera(cfg), cfg,
                   prop=PropagationOptions(pad2x=True))


def test_large_buckets_sorted_globally(gpu_ctx, oracle):
    # the reference's own bench scene packs thousands of splats into a few tiles
    # (holo_main.cpp:53-81): exercises buckets above the in-CTA sort capacity
    cfg = WaveConfig(nx=64, ny=64, wavelengths=RGB, num_planes=2)
    s = synthetic_scene(6000, cfg, 26)
    s.positions[:, :2] *= 0.05
    g, r, _ = check_pipeline(gpu_ctx, oracle, s, wide_camera(cfg), cfg)
    assert int(np.diff(r.raster.bucket_start.astype(np.int64)).max()) > 1024


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_tiled_equals_brute_force_bitwise_without_termination(gpu_ctx, oracle, seed):
    """test_rasterizer.cpp:244-255 on the GPU: with term_eps = 0 the tiled raster
    (bucket lists, accept-box culling) equals the untiled brute force bit for bit;
    the brute force itself matches the reference's (rasterizer.cpp:265-315)."""
    cfg = desk_config(48, 2)
    cam = front_camera(cfg)
    st = RenderSettings(term_eps=0.0)
    s = random_scene(30, cfg, seed)
    tiled = api.raster_forward(s, cam, cfg, st, ctx=gpu_ctx).layers
    brute = api.brute_force_forward(s, cam, cfg, st, ctx=gpu_ctx)
    for l in range(cfg.num_planes):
        assert np.array_equal(np.asarray(tiled[l]), brute[l])
    ref = oracle.brute_force_forward(s, cam, cfg, st)
    assert rel_l2(np.stack(brute), ref[:, :cfg.channels()]) <= 1e-5


def test_brute_force_soft_assignment_and_dense_overlap(gpu_ctx, oracle):
    cfg = WaveConfig(nx=64, ny=48, wavelengths=RGB, num_planes=3)
    for st, s in ((RenderSettings(term_eps=0.0, soft_assignment=True, soft_tau=1.0), synthetic_scene(300, cfg, 33)),
                  (RenderSettings(term_eps=0.0), overlapping_scene(200, cfg, 34))):
        cam = wide_camera(cfg) if st.soft_assignment else front_camera(cfg)
        tiled = api.raster_forward(s, cam, cfg, st, ctx=gpu_ctx).layers
        brute = api.brute_force_forward(s, cam, cfg, st, ctx=gpu_ctx)
        assert np.array_equal(np.stack(tiled), np.stack(brute))
        ref = oracle.brute_force_forward(s, cam, cfg, st)
        assert rel_l2(np.stack(brute), ref[:, :cfg.channels()]) <= 1e-5


def test_render_is_deterministic(gpu_ctx):
    cfg = WaveConfig(nx=256, ny=192, wavelengths=RGB, num_planes=4)
    s = synthetic_scene(30000, cfg, 27)
    a = api.pipeline_forward(s, wide_camera(cfg), cfg, ctx=gpu_ctx)
    b = api.pipeline_forward(s, wide_camera(cfg), cfg, ctx=gpu_ctx)
    assert np.array_equal(a.hologram, b.hologram)
    assert np.array_equal(np.stack(a.intensities), np.stack(b.intensities))
    assert np.array_equal(a.raster.entries, b.raster.entries)


# ---------------------------------------------------------------- rasterizer KATs (test_rasterizer.cpp) on the GPU

def centred(n, logits, phases=None):
    cfg = desk_config(32, 1)
    cam = front_camera(cfg)
    z = 0.3
    off = 0.5 * z / cam.focal_px
    s = single_scene(n, 1)
    s.positions = np.tile([off, off, z], (n, 1))
    s.log_scales = np.full((n, 3), np.log(0.004))
    s.amplitudes = np.ones((n, 3))
    s.opacity_logits = np.array(logits, dtype=float)
    if phases is not None:
        s.phases = np.array(phases, dtype=float)
    return cfg, cam, s


def test_blending_kats(gpu_ctx):
    # test_rasterizer.cpp:117-157, fp32 tolerance
    cfg, cam, s = centred(1, [math.log(0.8 / 0.2)])
    r = api.raster_forward(s, cam, cfg, ctx=gpu_ctx)
    assert abs(r.layers[0][0, 16, 16] - 0.8) < 1e-6 and abs(r.t_final[0, 16, 16] - 0.2) < 1e-6
    cfg, cam, s = centred(1, [math.log(0.8 / 0.2)], [[math.pi / 2] * 3])
    assert abs(api.raster_forward(s, cam, cfg, ctx=gpu_ctx).layers[0][0, 16, 16] - 0.8j) < 1e-6
    cfg, cam, s = centred(2, [0.0, 0.0], [[0, 0, 0], [math.pi] * 3])
    r = api.raster_forward(s, cam, cfg, ctx=gpu_ctx)
    assert abs(r.layers[0][0, 16, 16] - 0.25) < 1e-6 and abs(r.t_final[0, 16, 16] - 0.25) < 1e-6


def test_equal_depth_tie_by_index(gpu_ctx):
    cfg = desk_config(32, 1)
    s = single_scene(2, 1)
    s.positions = np.array([[0.0, 0.0, 0.3], [0.0, 0.0, 0.3]])
    s.log_scales = np.full((2, 3), np.log(0.005))
    s.amplitudes = np.ones((2, 3))
    s.phases = np.array([[0.0] * 3, [math.pi / 2] * 3])
    r = api.raster_forward(s, front_camera(cfg), cfg, ctx=gpu_ctx)
    first_bucket = r.entries["bucket"][0]
    assert list(r.entries["gidx"][r.entries["bucket"] == first_bucket]) == [0, 1]


@pytest.mark.parametrize("n", [20, 50, 100, 200])
def test_depths_equal_in_fp32_sort_by_f64_depth(gpu_ctx, n):
    """Bucket order is (zc, gidx) (rasterizer.cpp:221-224) even where distinct f64
    depths round to one fp32 value (the warp sort's fast key) and gidx runs against
    depth: warp-sorted bucket sizes of <= 32, <= 64, <= 128 and <= 256 entries."""
    cfg = desk_config(32, 1)
    s = single_scene(n, 1)
    s.positions = np.array([[0.0, 0.0, 0.3 + 1e-12 * (n - i)] for i in range(n)])
    s.log_scales = np.full((n, 3), np.log(0.005))
    s.amplitudes = np.ones((n, 3))
    r = api.raster_forward(s, front_camera(cfg), cfg, ctx=gpu_ctx)
    first_bucket = r.entries["bucket"][0]
    sel = r.entries["bucket"] == first_bucket
    depth, gidx = r.entries["depth"][sel], r.entries["gidx"][sel]
    assert len(gidx) == n
    assert len(np.unique(np.float32(depth))) < n  # the fp32 keys do collide
    order = sorted(range(n), key=lambda k: (depth[k], gidx[k]))
    assert list(order) == list(range(n))
    assert list(gidx) == sorted(gidx, key=lambda g: (r.projected["zc"][g], g))


@pytest.mark.parametrize("n", [20, 50, 100, 200])
def test_depths_apart_in_fp32_but_equal_in_the_short_key(gpu_ctx, n):
    """Depths two fp32 ulps apart: distinct fp32 keys, but equal 32-bit short keys
    (fp32 depth without its low mantissa bits), so the sort must detect the shared
    short key and fall back; gidx runs against depth."""
    cfg = desk_config(32, 1)
    s = single_scene(n, 1)
    ulp = float(np.spacing(np.float32(0.3)))
    s.positions = np.array([[0.0, 0.0, 0.3 + 2 * ulp * (n - i)] for i in range(n)])
    s.log_scales = np.full((n, 3), np.log(0.005))
    s.amplitudes = np.ones((n, 3))
    r = api.raster_forward(s, front_camera(cfg), cfg, ctx=gpu_ctx)
    first_bucket = r.entries["bucket"][0]
    sel = r.entries["bucket"] == first_bucket
    gidx = r.entries["gidx"][sel]
    assert len(gidx) == n
    zc = r.projected["zc"]
    assert len(np.unique(np.float32(zc[gidx]))) == n  # the fp32 keys do not collide
    assert list(gidx) == sorted(gidx, key=lambda g: (zc[g], g))
    assert list(gidx) == list(range(n - 1, -1, -1))


def test_culling_and_clamp(gpu_ctx):
    cfg = desk_config(32, 1)
    s = single_scene(2, 1)
    s.positions = np.array([[0.0, 0.0, 1e-4], [0.0, 0.0, -0.5]])
    s.log_scales = np.full((2, 3), np.log(0.005))
    s.amplitudes = np.ones((2, 3))
    s.opacity_logits = np.array([2.0, 2.0])
    r = api.raster_forward(s, front_camera(cfg), cfg, ctx=gpu_ctx)
    assert list(r.projected["valid"]) == [0, 0] and not np.any(np.stack(r.layers))
    s = single_scene(1, 1)
    s.positions = np.array([[0.0, 0.0, 0.3]])
    s.log_scales = np.full((1, 3), np.log(0.05))
    s.amplitudes = np.ones((1, 3))
    s.opacity_logits = np.array([40.0])
    r = api.raster_forward(s, front_camera(cfg), cfg, ctx=gpu_ctx)
    assert r.t_final[0, 16, 16] >= 1.0 - 0.999 - 1e-7
    assert np.abs(np.stack(r.layers)).max() <= 0.999 + 1e-6


def test_rejects_bad_inputs(gpu_ctx):
    cfg = desk_config(32, 2)
    s = random_scene(3, cfg, 1)
    bad = front_camera(cfg)
    bad.width = 16
    with pytest.raises(HoloError):
        api.raster_forward(s, bad, cfg, ctx=gpu_ctx)
    s.rotations[1] = 0.0  # degenerate quaternion: validated on the device (scene.cpp:27)
    gpu_ctx.upload_scene(s)
    with pytest.raises(HoloError) as e:
        gpu_ctx.render(front_camera(cfg), cfg)
    assert e.value.kind == "config" and "quaternion" in str(e.value)
    s = random_scene(3, cfg, 1)
    s.amplitudes[0, 0] = -1.0
    gpu_ctx.upload_scene(s)
    with pytest.raises(HoloError):
        gpu_ctx.render(front_camera(cfg), cfg)


# ---------------------------------------------------------------- asynchronous frames (holo_ctx_set_async)

def _frame(ctx, C, H, W, L_):
    holo = ctx.download(L.BUF_HOLOGRAM, np.complex64, (C, H, W))
    ints = ctx.download(L.BUF_INTENSITY, np.float32, (L_, C, H, W))
    return holo, ints


def test_async_frames_equal_sync_frames():
    cfg = WaveConfig(nx=256, ny=192, wavelengths=RGB, num_planes=4)
    scenes = [synthetic_scene(20000, cfg, 40 + i) for i in range(3)]
    cam = wide_camera(cfg)
    ctx = api.Context(0, use_torch_stream=False)
    want, infos = [], []
    for s in scenes:
        ctx.upload_scene(s)
        infos.append((ctx.render(cam, cfg).num_entries, ctx.info.max_bucket, ctx.info.num_valid))
        want.append(_frame(ctx, 3, 192, 256, 4))
    ctx.set_async(True)
    for s, w, inf in zip(scenes, want, infos):
        ctx.upload_scene(s)
        assert ctx.render(cam, cfg).num_entries == 0  # not known until frame_status
        st = ctx.frame_status()
        assert (st.num_entries, st.max_bucket, st.num_valid) == inf
        got = _frame(ctx, 3, 192, 256, 4)
        assert np.array_equal(got[0], w[0]) and np.array_equal(got[1], w[1])
    # lists of an asynchronous frame (E read back lazily)
    ctx.render(cam, cfg, outputs=L.OUT_HOLOGRAM | L.OUT_LISTS)
    p, nbytes = ctx.buffer(L.BUF_ENTRY_GIDX)
    assert nbytes == 4 * infos[-1][0]
    ctx.close()


def test_async_capacity_and_validation_reported_by_frame_status():
    cfg = WaveConfig(nx=128, ny=128, wavelengths=RGB, num_planes=2)
    s = synthetic_scene(5000, cfg, 44)
    cam = wide_camera(cfg)
    ctx = api.Context(0, use_torch_stream=False)
    ctx.set_async(True)
    ctx.upload_scene(s)
    with pytest.raises(HoloError) as e:  # nothing reserved and no synchronous frame yet
        ctx.render(cam, cfg)
    assert e.value.kind == "config"
    ctx.reserve_entries(100)
    ctx.render(cam, cfg)  # overflows: dropped entries, no out-of-bounds access
    with pytest.raises(HoloError) as e:
        ctx.frame_status()
    assert e.value.kind == "numeric" and "reserve" in str(e.value)
    ctx.render(cam, cfg)  # the failed status grew the reservation
    E = ctx.frame_status().num_entries
    ctx.set_async(False)
    assert ctx.render(cam, cfg).num_entries == E
    ref = _frame(ctx, 3, 128, 128, 2)
    ctx.set_async(True)
    ctx.render(cam, cfg)
    ctx.frame_status()
    got = _frame(ctx, 3, 128, 128, 2)
    assert np.array_equal(got[0], ref[0])
    bad = random_scene(3, cfg, 1)
    bad.amplitudes[0, 0] = -1.0
    ctx.upload_scene(bad)
    ctx.render(cam, cfg)
    with pytest.raises(HoloError) as e:
        ctx.frame_status()
    assert e.value.kind == "config" and "non-negative" in str(e.value)
    ctx.frame_status()  # flags cleared
    ctx.close()


def test_async_overflow_with_large_buckets_and_backward_rejected():
    # a heavily overflowed asynchronous frame: many buckets above the in-CTA sort
    # capacity (1024) while only 100 entries are reserved.  The large-bucket list
    # is bounded by the clamped capacity, and a backward on the truncated lists
    # is refused instead of running past its per-entry gradient buffer.
    import torch

    cfg = WaveConfig(nx=64, ny=64, wavelengths=RGB, num_planes=2)
    s = overlapping_scene(40000, cfg, 45)
    s.positions[:, :2] *= 0.2  # every Gaussian covers most of the 16 tiles
    cam = wide_camera(cfg)
    ctx = api.Context(0, use_torch_stream=False)
    ctx.upload_scene(s)
    info = ctx.render(cam, cfg, outputs=L.OUT_HOLOGRAM | L.OUT_INTENSITY | L.OUT_AUX)
    assert info.max_bucket > 1024 and info.num_entries > 20 * 1025
    ref = _frame(ctx, 3, 64, 64, 2)
    ctx.close()
    ctx = api.Context(0, use_torch_stream=False)  # no synchronous frame sized its entry buffers
    ctx.upload_scene(s)
    ctx.set_async(True)
    ctx.reserve_entries(100)
    ctx.render(cam, cfg, outputs=L.OUT_HOLOGRAM | L.OUT_INTENSITY | L.OUT_AUX)
    gl = torch.zeros((2, 3, 64, 64), dtype=torch.complex64, device="cuda:0")
    with pytest.raises(HoloError) as e:
        ctx.raster_backward(cam, cfg, None, gl, s.size())
    assert "overflowed" in str(e.value)
    with pytest.raises(HoloError) as e:
        ctx.frame_status()
    assert e.value.kind == "numeric" and "reserve" in str(e.value)
    ctx.render(cam, cfg, outputs=L.OUT_HOLOGRAM | L.OUT_INTENSITY | L.OUT_AUX)  # the reservation grew
    assert ctx.frame_status().num_entries == info.num_entries
    got = _frame(ctx, 3, 64, 64, 2)
    assert np.array_equal(got[0], ref[0])
    ctx.raster_backward(cam, cfg, None, gl, s.size())
    ctx.close()


def test_async_upload_render_download_pipeline():
    # scene uploads on the copy-in stream into the set the running frame does not
    # read, downloads on the copy-out stream: several frames enqueued back to back
    # must each see their own scene and land in their own host buffers
    import torch

    cfg = WaveConfig(nx=256, ny=192, wavelengths=RGB, num_planes=4)
    scenes = [synthetic_scene(15000, cfg, 50 + i) for i in range(4)]
    cam = wide_camera(cfg)
    ctx = api.Context(0, use_torch_stream=False)
    want = []
    for s in scenes:
        ctx.upload_scene(s)
        ctx.render(cam, cfg)
        want.append(_frame(ctx, 3, 192, 256, 4))
    ctx.set_async(True)
    pins = []
    for s in scenes:
        arrs = [torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).pin_memory() for a in
                (s.positions, s.rotations, s.log_scales, s.amplitudes, s.opacity_logits, s.phases, s.plane_logits)]
        pins.append(arrs)
    outs = [(torch.empty((3, 192, 256), dtype=torch.complex64).pin_memory(),
             torch.empty((4, 3, 192, 256), dtype=torch.float32).pin_memory()) for _ in scenes]
    for rep in range(2):
        for s, arrs, (hh, ih) in zip(scenes, pins, outs):
            ctx.upload_scene_pointers(s.size(), 4, [a.data_ptr() for a in arrs], device=False)
            ctx.render(cam, cfg)
            ctx.download_into(L.BUF_HOLOGRAM, hh.data_ptr(), hh.numel() * 8, wait=False)
            ctx.download_into(L.BUF_INTENSITY, ih.data_ptr(), ih.numel() * 4, wait=False)
        ctx.synchronize()
        ctx.frame_status()
        for w, (hh, ih) in zip(want, outs):
            assert np.array_equal(hh.numpy(), w[0]) and np.array_equal(ih.numpy(), w[1])
    ctx.close()


def test_two_async_contexts_overlap_and_agree():
    import torch

    cfg = WaveConfig(nx=256, ny=256, wavelengths=RGB, num_planes=4)
    s = synthetic_scene(30000, cfg, 45)
    cam = wide_camera(cfg)
    ctxs = [api.Context(0, use_torch_stream=False) for _ in range(2)]
    for c in ctxs:
        c.upload_scene(s)
        c.render(cam, cfg)
        c.set_async(True)
    ref = _frame(ctxs[0], 3, 256, 256, 4)
    for _ in range(4):
        for c in ctxs:
            c.render(cam, cfg)
    for c in ctxs:
        c.frame_status()
        got = _frame(c, 3, 256, 256, 4)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
        c.close()
    torch.cuda.synchronize()


# ---------------------------------------------------------------- plane sharding (begin / all-reduce / end) on one GPU

def test_plane_sharded_halves_equal_full_render(gpu_ctx):
    import torch

    cfg = WaveConfig(nx=256, ny=256, wavelengths=RGB, num_planes=4)
    s = synthetic_scene(20000, cfg, 31)
    cam = wide_camera(cfg)
    full = api.pipeline_forward(s, cam, cfg, ctx=gpu_ctx, raster=False)
    gpu_ctx.upload_scene(s)
    C, H, W = 3, 256, 256
    spec = torch.zeros((C, H, W, 2), dtype=torch.float32, device="cuda")
    parts = []
    for pb, pe in [(0, 2), (2, 4)]:  # two "ranks" emulated in sequence; the all-reduce is a sum
        part = torch.empty_like(spec)
        gpu_ctx.render_begin(cam, cfg, None, None, pb, pe, part.data_ptr(), 0)
        torch.cuda.synchronize()
        parts.append(part)
    spec = parts[0] + parts[1]
    torch.cuda.synchronize()
    ints = []
    for pb, pe in [(0, 2), (2, 4)]:
        outs = L.OUT_INTENSITY | (L.OUT_HOLOGRAM if pb == 0 else 0)
        gpu_ctx.render_end(cfg, None, pb, pe, spec.data_ptr(), outs)
        ints.append(gpu_ctx.download(L.BUF_INTENSITY, np.float32, (pe - pb, C, H, W)))
        if pb == 0:
            holo = gpu_ctx.download(L.BUF_HOLOGRAM, np.complex64, (C, H, W))
    assert rel_l2(holo, full.hologram) < 1e-5
    assert rel_l2(np.concatenate(ints), np.stack(full.intensities)) < 1e-5


# ---------------------------------------------------------------- BASELINE configurations at full size

def _bucket_sizes(bucket_start):
    return np.diff(np.asarray(bucket_start, dtype=np.int64))


def _rel_l2_chunked(gpu_planes, ref):
    """rel-L2 over a plane stack without materialising full-size differences
    (C5 layers are 6.4 GB in f64)."""
    num = den = 0.0
    for l in range(ref.shape[0]):
        r = ref[l]
        g = np.asarray(gpu_planes[l])[: r.shape[0]]
        num += float(np.sum(np.abs(g.astype(r.dtype) - r) ** 2))
        den += float(np.sum(np.abs(r) ** 2))
    return math.sqrt(num / den) if den > 0 else math.sqrt(num)


def check_baseline_frame(ctx, ora, scene, cam, cfg):
    """Full-size frame parity at the BASELINE bars: layers, hologram and
    intensities rel-L2 <= 1e-4, per-plane PSNR within 0.01 dB, lists bit-exact."""
    C = cfg.channels()
    g = api.pipeline_forward(scene, cam, cfg, ctx=ctx, replayed=False)
    r = ora.pipeline_forward(scene, cam, cfg, replayed=False)
    assert np.array_equal(g.raster.bucket_start, r.raster.bucket_start)
    assert np.array_equal(g.raster.entries["gidx"], r.raster.entry_gidx)
    assert _rel_l2_chunked(g.raster.layers, r.raster.layers[:, :C]) <= 1e-4
    assert rel_l2(g.hologram, r.hologram) <= 1e-4
    assert _rel_l2_chunked(g.intensities, r.intensities) <= 1e-4
    for l in range(cfg.num_planes):
        t = 0.9025 * r.intensities[l]
        assert abs(psnr(np.asarray(g.intensities[l]), t) - psnr(r.intensities[l], t)) <= 0.01
    return g, r


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_baseline_config_parity(gpu_ctx, oracle, name):
    c = CONFIGS[name]
    cfg = c.wave()
    g, r = check_baseline_frame(gpu_ctx, oracle, synthetic_scene(c.n, cfg, c.seed), c.cameras()[0], cfg)
    if name == "C3":  # every bucket takes the warp-per-bucket sort (<= 256 entries)
        assert 0 < _bucket_sizes(r.raster.bucket_start).max() <= 256


@pytest.mark.slow
@pytest.mark.parametrize("view", [0, 63])
def test_baseline_c4_views_parity(gpu_ctx, oracle, view):
    """C4 (1M Gaussians, 1024x1024, 6 planes, RGB): the two extreme views of the
    64-view batch (yaw -0.1 and +0.1 rad) at full size.  C4's density puts
    thousands of buckets above 128 entries: the warp sort's widest (eight keys per
    lane) network."""
    c = CONFIGS["C4"]
    cfg = c.wave()
    scene = synthetic_scene(c.n, cfg, c.seed)
    g, r = check_baseline_frame(gpu_ctx, oracle, scene, c.cameras()[view], cfg)
    sizes = _bucket_sizes(r.raster.bucket_start)
    assert (sizes > 128).sum() > 1000 and sizes.max() <= 256


@pytest.mark.slow
def test_baseline_c5_parity(ref_oracle):
    """C5 (3M Gaussians, 3840x2160, 16 planes, RGB; 9.6M entries): the 3840- and
    2160-point static plans, the one-row-per-CTA row pass and the 16-plane
    spectrum, checked against the reference build itself (oracle/_ref; about a
    minute on the box's host cores and 25 GB of host memory)."""
    c = CONFIGS["C5"]
    cfg = c.wave()
    ctx = api.Context(0)
    check_baseline_frame(ctx, ref_oracle, synthetic_scene(c.n, cfg, c.seed), c.cameras()[0], cfg)
    ctx.close()


@pytest.mark.parametrize("W,H", [(2048, 2160), (3840, 2048)])
def test_static_plan_sizes(gpu_ctx, oracle, W, H):
    """The 2048-, 2160- and 3840-point compile-time plans as both the row and
    the column transform of the render path (a small scene on a large grid)."""
    cfg = WaveConfig(nx=W, ny=H, wavelengths=RGB, num_planes=2)
    check_pipeline(gpu_ctx, oracle, synthetic_scene(20000, cfg, 31), wide_camera(cfg), cfg)


def test_every_sort_path_in_one_frame(gpu_ctx, oracle):
    """One frame whose buckets take all three bucket sorts: the warp bitonic
    (<= 256 entries), the in-CTA sort of the compositing CTA (257..1024) and the
    device-wide sort of k_sort_large_dev (> 1024)."""
    cfg = WaveConfig(nx=128, ny=128, wavelengths=RGB, num_planes=2)
    s = synthetic_scene(12000, cfg, 32)
    s.positions[:4000, :2] *= 0.03   # a dense core: buckets above 1024
    s.positions[4000:8000, :2] *= 0.4
    g, r, _ = check_pipeline(gpu_ctx, oracle, s, wide_camera(cfg), cfg)
    sizes = _bucket_sizes(r.raster.bucket_start)
    assert (sizes > 1024).any() and ((sizes > 256) & (sizes <= 1024)).any() and ((sizes > 0) & (sizes <= 256)).any()


def test_plane_subset_shards_render_the_same_layers(gpu_ctx):
    """sharding.plane_subset: a rank holding only its planes' Gaussians renders the
    full scene's partial spectrum for those planes bit for bit (hard assignment:
    one plane per Gaussian; an order-preserving subset keeps every bucket's order)."""
    import torch

    from paper_2506_08350_b200.sharding import plane_ranges, plane_subset

    cfg = WaveConfig(nx=256, ny=256, wavelengths=RGB, num_planes=4)
    s = synthetic_scene(20000, cfg, 31)
    cam = wide_camera(cfg)
    C, H, W = 3, 256, 256
    for pb, pe in plane_ranges(4, 2):
        full_part = torch.empty((C, H, W, 2), dtype=torch.float32, device="cuda")
        gpu_ctx.upload_scene(s)
        gpu_ctx.render_begin(cam, cfg, None, None, pb, pe, full_part.data_ptr(), 0)
        sub = plane_subset(s, pb, pe)
        assert 0 < sub.size() < s.size()
        sub_part = torch.empty_like(full_part)
        gpu_ctx.upload_scene(sub)
        gpu_ctx.render_begin(cam, cfg, None, None, pb, pe, sub_part.data_ptr(), 0)
        torch.cuda.synchronize()
        assert torch.equal(full_part, sub_part)

def test_plane_assignment_follows_the_strict_scan(gpu_ctx):
    """The device's hard plane (ste_assign's argmax, scene.cpp:132-152) equals the
    reference's strict-'>' scan from plane 0 -- first index of the largest logit,
    NaNs never win, a NaN logit 0 keeps plane 0, -0.0 ties +0.0 -- for Gaussians in
    full shared-memory slices and in the tail slice (read from global memory)."""
    cfg = desk_config(32, 5)
    n = 150
    rng = np.random.default_rng(11)
    s = random_scene(n, cfg, 12)
    lg = rng.integers(-2, 3, size=(n, 5)).astype(np.float64)  # many exact ties
    lg[::7, 0] = np.nan
    lg[3::11, 2] = np.nan
    lg[5::13] = np.nan
    lg[6::17, 1] = -0.0
    lg[6::17, 3] = 0.0
    lg[8::19, 4] = np.inf
    lg[9::23, 0] = -np.inf
    s.plane_logits = lg
    r = api.raster_forward(s, front_camera(cfg), cfg, ctx=gpu_ctx)

    def scan(row):
        best = 0
        for l in range(1, len(row)):
            if row[l] > row[best]:
                best = l
        return best

    assert list(r.projected["plane"]) == [scan(row) for row in lg]
