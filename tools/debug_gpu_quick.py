"""Quick GPU bring-up script (not a pytest module): prints parity numbers per stage."""
import sys, os, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
import numpy as np
from oracle.oracle import Oracle, rel_l2
from paper_2506_08350_b200 import api
from paper_2506_08350_b200.holotypes import WaveConfig, PropagationOptions
from paper_2506_08350_b200.scenes import synthetic_scene, front_camera

ora = Oracle("restate")
ctx = api.Context(0)
rng = np.random.default_rng(0)
def step(name, f):
    try:
        t = time.time(); r = f(); print(f"[{name}] {r}  ({time.time()-t:.2f}s)", flush=True)
    except Exception:
        print(f"[{name}] FAILED"); traceback.print_exc()

for (h, w) in [(48, 64), (17, 13), (256, 256), (1080, 1920), (30, 42)]:
    x = rng.standard_normal((2, h, w)) + 1j * rng.standard_normal((2, h, w))
    step(f"fft2 f64 {w}x{h}", lambda: rel_l2(ctx.fft2(x, False, "f64"), np.fft.fft2(x)))
    step(f"fft2 f32 {w}x{h}", lambda: rel_l2(ctx.fft2(x, False, "f32"), np.fft.fft2(x)))
    step(f"ifft2 f64 {w}x{h}", lambda: rel_l2(ctx.fft2(x, True, "f64"), np.fft.ifft2(x)))

cfg = WaveConfig(nx=64, ny=48, num_planes=3)
u = rng.standard_normal((3, 48, 64)) + 1j * rng.standard_normal((3, 48, 64))
for prec in ("f64", "f32"):
    for z in (1.7e-3, -2e-3, 0.0):
        step(f"propagate {prec} z={z}", lambda: rel_l2(ctx.propagate(u, cfg, z, None, prec), ora.propagate(u, cfg, z)))
    step(f"propagate pad {prec}", lambda: rel_l2(ctx.propagate(u, cfg, 1e-3, PropagationOptions(pad2x=True), prec), ora.propagate(u, cfg, 1e-3, PropagationOptions(pad2x=True))))
    step(f"propagate local {prec}", lambda: rel_l2(ctx.propagate(u, cfg, 50e-3, PropagationOptions(local_band_limit=True), prec), ora.propagate(u, cfg, 50e-3, PropagationOptions(local_band_limit=True))))
    step(f"tf {prec}", lambda: rel_l2(ctx.transfer_function(cfg, 1.3e-3, None, prec), ora.transfer_function(cfg, 1.3e-3)))

for (n, W, H, L, wl) in [(300, 64, 48, 3, (639e-9, 532e-9, 473e-9)), (3000, 256, 256, 3, (515e-9,)), (20000, 512, 384, 4, (638e-9, 520e-9, 450e-9))]:
    cfg = WaveConfig(nx=W, ny=H, wavelengths=wl, num_planes=L)
    sc = synthetic_scene(n, cfg, 5)
    cam = front_camera(cfg)
    def run():
        g = api.pipeline_forward(sc, cam, cfg, ctx=ctx)
        r = ora.pipeline_forward(sc, cam, cfg)
        gl = np.stack(g.raster.layers); rl = r.raster.layers[:, :len(wl)]
        out = dict(E=len(g.raster.entries), E_ref=len(r.raster.entry_gidx),
                   lists=bool(np.array_equal(g.raster.entries["gidx"], r.raster.entry_gidx)),
                   bstart=bool(np.array_equal(g.raster.bucket_start, r.raster.bucket_start)),
                   layers=rel_l2(gl, rl), holo=rel_l2(g.hologram, r.hologram),
                   rep=rel_l2(np.stack(g.replayed), r.replayed), ints=rel_l2(np.stack(g.intensities), r.intensities),
                   ncontrib_mismatch=int((g.raster.n_contrib != r.raster.n_contrib).sum()))
        for k in ("mu_x", "mu_y", "inv00", "inv01", "inv11", "radius", "zc", "alpha_sig", "valid", "plane"):
            out["proj_" + k] = bool(np.array_equal(g.raster.projected[k], r.raster.projected[k]))
        return out
    step(f"render n={n} {W}x{H} L={L} C={len(wl)}", run)
print("launches", ctx.launch_count())
