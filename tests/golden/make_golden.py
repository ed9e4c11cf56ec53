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
        # (deterministic: re-running reproduces the committed files bit for bit)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(name, os.path.getsize(path), "bytes, E =", len(r.raster.entry_gidx))


if __name__ == "__main__":
    main()
