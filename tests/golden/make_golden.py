"""Generate tests/golden/*.npz from the reference itself.

Runs holo::pipeline_forward / raster_forward of the reference C++ sources
(/root/reference/proj/src compiled in place by oracle/Makefile into oracle/_ref,
called through oracle/ref_capi.cpp) on small deterministic scenes and stores
inputs and outputs.  The reference ships no golden vectors, so these
fixtures are what pins the CPU restatement and the GPU path on the GPU box, where
/root/reference does not exist.

    python tests/golden/make_golden.py        # needs oracle/_ref (make -C oracle ref)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from conftest import mild_posed_camera, overlapping_scene  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2506_08350_b200.holotypes import CameraView, PropagationOptions, RenderSettings, WaveConfig  # noqa: E402
from paper_2506_08350_b200.scenes import front_camera, synthetic_scene  # noqa: E402

RGB = (639e-9, 532e-9, 473e-9)
TL_KEYS = ("recon", "ssim", "opacity", "total", "psnr_mean")
OPT_CFG = (0.01, 0.001, 0.005, 0.0025, 0.0025, 0.025, 0.01, 0.9, 0.99, 0.99, 1e-8, 1e-5)
GROUPS = ("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases", "plane_logits")


def training_golden(ref):
    """losses.cpp on seeded stacks and optimizer_step runs (Adan and Adam, a
    non-finite step skipped) from fresh moments -> training.npz."""
    rng = np.random.default_rng(300)
    I = rng.random((2, 3, 20, 24))
    G = np.clip(I + 0.2 * rng.standard_normal(I.shape), 0.0, 1.0)
    M = (rng.random((2, 20, 24)) > 0.5).astype(np.float64)
    out = dict(ls_I=I, ls_G=G, ls_M=M)
    for plain in (0, 1):
        r, s, ps, g = ref.losses(I, G, M, lambda_ssim=0.2, plain=bool(plain))
        out.update({f"ls{plain}_recon": r, f"ls{plain}_ssim": s, f"ls{plain}_psnr": ps, f"ls{plain}_grad": g})
    cfg = WaveConfig(nx=48, ny=48, wavelengths=RGB, num_planes=3)
    scene = synthetic_scene(50, cfg, 16)
    steps = []
    for k in range(5):
        gr = np.random.default_rng(400 + k)
        steps.append({n: gr.standard_normal(np.shape(getattr(scene, n))) for n in GROUPS})
    steps[2]["phases"][3, 1] = np.inf
    out.update(op_num_planes=scene.num_planes, **{f"op_scene_{n}": getattr(scene, n) for n in GROUPS},
               **{f"op_g{k}_{n}": steps[k][n] for k in range(5) for n in GROUPS}, op_cfg=np.array(OPT_CFG))
    for adam in (0, 1):
        want, applied = ref.optimizer_run(scene, steps, OPT_CFG, use_adam=bool(adam), schedule_total=3)
        out.update({f"op{adam}_applied": applied, **{f"op{adam}_{n}": want[n] for n in GROUPS}})
    # phase-only conversion (phase_only.cpp) of a rendered 32x32 hologram
    pcfg = WaveConfig(nx=32, ny=32, wavelengths=RGB, num_planes=2)
    P = ref.pipeline_forward(synthetic_scene(60, pcfg, 17), front_camera(pcfg), pcfg, RenderSettings(),
                             PropagationOptions()).hologram
    theta = np.angle(P) + np.random.default_rng(500).uniform(-0.3, 0.3, P.shape)
    pl, pg = ref.phase_only_loss(P, theta, pcfg)
    pphase, ptrace = ref.convert_phase_only(P, pcfg, 12, 0.05)
    out.update(po_P=P, po_theta=theta, po_loss=pl, po_grad=pg, po_phase=pphase, po_trace=ptrace)
    path = os.path.join(HERE, "training.npz")
    np.savez_compressed(path, **out)
    print("training", os.path.getsize(path), "bytes")


def cases():
    cfg = WaveConfig(nx=48, ny=40, wavelengths=(515e-9,), num_planes=3)
    yield "c1_mini", synthetic_scene(150, cfg, 11), front_camera(cfg), cfg, RenderSettings(), PropagationOptions()
    cfg = WaveConfig(nx=64, ny=48, wavelengths=RGB, num_planes=2)
    cam = mild_posed_camera(cfg)
    cam.focal_px = 64.0
    yield "rgb_posed", synthetic_scene(300, cfg, 12), cam, cfg, RenderSettings(), PropagationOptions()
    cfg = WaveConfig(nx=40, ny=40, wavelengths=RGB, num_planes=3)
    yield ("tile8_soft", synthetic_scene(120, cfg, 13), front_camera(cfg), cfg,
           RenderSettings(tile=8, soft_assignment=True), PropagationOptions())
    cfg = WaveConfig(nx=32, ny=32, wavelengths=RGB, num_planes=2)
    yield ("dense_overlap", overlapping_scene(40, cfg, 14), CameraView(focal_px=150.0, width=32, height=32), cfg,
           RenderSettings(), PropagationOptions())
    cfg = WaveConfig(nx=48, ny=48, wavelengths=RGB, num_planes=2)
    yield "pad2x", synthetic_scene(100, cfg, 15), front_camera(cfg), cfg, RenderSettings(), PropagationOptions(
        pad2x=True)


def main():
    ref = Oracle("ref")
    for name, scene, cam, cfg, st, prop in cases():
        r = ref.pipeline_forward(scene, cam, cfg, st, prop)
        out = dict(
            positions=scene.positions, rotations=scene.rotations, log_scales=scene.log_scales,
            amplitudes=scene.amplitudes, opacity_logits=scene.opacity_logits, phases=scene.phases,
            plane_logits=scene.plane_logits, num_planes=scene.num_planes,
            cam_pose=np.array(cam.pose, dtype=float), cam_focal=cam.focal_px, cam_cx=cam.cx, cam_cy=cam.cy,
            nx=cfg.nx, ny=cfg.ny, pitch=cfg.pitch, wavelengths=np.array(cfg.wavelengths), distance=cfg.distance,
            volume_depth=cfg.volume_depth,
            st_tile=st.tile, st_soft=int(st.soft_assignment), pad2x=int(prop.pad2x),
            hologram=r.hologram, intensities=r.intensities, layers=r.raster.layers,
            t_final=r.raster.t_final, n_contrib=r.raster.n_contrib, entry_gidx=r.raster.entry_gidx,
            entry_bucket=r.raster.entry_bucket, bucket_start=r.raster.bucket_start,
            mu_x=r.raster.projected["mu_x"], mu_y=r.raster.projected["mu_y"], zc=r.raster.projected["zc"],
        )
        if cfg.channels() == 3:
            # the gradient branch of total_loss (pipeline.cpp:63-80) for a seeded dL/dI
            gi = np.random.default_rng(100 + len(name)).standard_normal(r.intensities.shape)
            grads, gh, gl = ref.pipeline_backward(scene, cam, cfg, st, prop, gi)
            out.update(bwd_gi=gi, bwd_gholo=gh, bwd_glayers=gl, **{f"bwd_{k}": v for k, v in grads.items()})
            # total_loss (pipeline.cpp:30-95) against a seeded focal-stack target
            rng = np.random.default_rng(200 + len(name))
            tgt = 0.5 * rng.random(r.intensities.shape)
            msk = (rng.random((cfg.num_planes, cfg.ny, cfg.nx)) > 0.6).astype(np.float64)
            bd, ps, tg = ref.total_loss(scene, cam, cfg, st, prop, tgt, msk, lambda_ssim=0.05, lambda_opacity=1e-2)
            out.update(tl_targets=tgt, tl_masks=msk, tl_breakdown=np.array([bd[k] for k in TL_KEYS]), tl_psnr=ps,
                       **{f"tl_{k}": v for k, v in tg.items()})
        # (deterministic: re-running reproduces the committed files bit for bit)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(name, os.path.getsize(path), "bytes, E =", len(r.raster.entry_gidx))
    training_golden(ref)


if __name__ == "__main__":
    main()
