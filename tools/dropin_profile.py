import os, subprocess, sys, tempfile
sys.path.insert(0, os.getcwd())
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene, write_scene
c = CONFIGS["C3"]; wave = c.wave()
with tempfile.TemporaryDirectory() as d:
    path = os.path.join(d, "s.holoscene")
    write_scene(path, synthetic_scene(c.n, wave, c.seed))
    cmd = ["paper_2506_08350_b200/lib/dropin_bench", path, "--nx", str(wave.nx), "--ny", str(wave.ny), "--planes", str(wave.num_planes),
           "--wavelengths", ",".join(repr(x) for x in wave.wavelengths), "--frames", "3", "--warmup", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, env=dict(os.environ, HOLO_DROPIN_PROFILE="1"))
    print(out.stdout[-500:]); print(out.stderr[-1500:])
