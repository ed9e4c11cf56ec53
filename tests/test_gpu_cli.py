"""The `holo` command-line front end (paper_2506_08350_b200/lib/holo, built from
cpp/holo_cli.cpp over the C++ drop-in): the render / propagate / bench
subcommands of the reference's holo_main.cpp, with its exit-code and JSON
conventions.  `propagate` must equal the in-process operator bit for bit
(test_cli.cpp:198-218)."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import rel_l2
from oracle.oracle import Oracle
from paper_2506_08350_b200 import api
from paper_2506_08350_b200.holotypes import PipelineOptions, WaveConfig
from paper_2506_08350_b200.scenes import front_camera, synthetic_scene, write_scene

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOLO = os.path.join(ROOT, "paper_2506_08350_b200", "lib", "holo")
MAGIC = b"HOLOFIELD" + b"\0" * 7


def write_field(path, f):
    c, h, w = f.shape
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(np.array([w, h, c], dtype="<u4").tobytes())
        fh.write(np.ascontiguousarray(f, dtype="<c16").tobytes())


def read_field(path):
    with open(path, "rb") as fh:
        assert fh.read(16) == MAGIC
        w, h, c = np.frombuffer(fh.read(12), dtype="<u4")
        return np.frombuffer(fh.read(), dtype="<c16").reshape(c, h, w)


def run(*args):
    if not os.path.exists(HOLO):
        pytest.skip("holo CLI not built")
    return subprocess.run([HOLO, *args], capture_output=True, text=True, timeout=300)


def test_propagate_matches_the_in_process_operator(tmp_path, gpu_ctx):
    rng = np.random.default_rng(9)
    u = rng.standard_normal((3, 32, 32)) + 1j * rng.standard_normal((3, 32, 32))
    write_field(tmp_path / "in.hfld", u)
    r = run("propagate", "--in", str(tmp_path / "in.hfld"), "--out", str(tmp_path / "out.hfld"), "--z-meters", "0.002")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["command"] == "propagate" and rep["energy_out"] == pytest.approx(rep["energy_in"], rel=1e-10)
    got = read_field(tmp_path / "out.hfld")
    cfg = WaveConfig(nx=32, ny=32, num_planes=1)
    assert np.array_equal(got, api.propagate(u, cfg, 0.002))  # bit for bit
    if Oracle.available("ref"):
        assert rel_l2(got, Oracle("ref").propagate(u, cfg, 0.002)) < 1e-12
    # one --wavelength per channel (holo_main.cpp:93-97): usage error, exit 2
    bad = run("propagate", "--in", str(tmp_path / "in.hfld"), "--out", str(tmp_path / "x.hfld"), "--z-meters",
              "0.002", "--wavelength", "532e-9")
    assert bad.returncode == 2 and "usage" in bad.stderr
    missing = run("propagate", "--in", str(tmp_path / "nope.hfld"), "--out", str(tmp_path / "x.hfld"), "--z-meters",
                  "0.002")
    assert missing.returncode == 1 and '"io"' in missing.stderr


def test_render_writes_the_pipeline_outputs(tmp_path, gpu_ctx):
    cfg = WaveConfig(nx=96, ny=64, num_planes=3)
    scene = synthetic_scene(2000, cfg, 5)
    write_scene(str(tmp_path / "s.holoscene"), scene)
    r = run("render", "--scene", str(tmp_path / "s.holoscene"), "--out-dir", str(tmp_path), "--nx", "96", "--ny", "64")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["gaussians"] == 2000 and rep["planes"] == 3 and rep["entries"] > 0
    out = api.pipeline_forward(scene, front_camera(cfg), cfg, PipelineOptions(), ctx=gpu_ctx)
    assert np.array_equal(read_field(tmp_path / "hologram.hfld"), out.hologram)
    for l in range(3):
        assert np.array_equal(read_field(tmp_path / f"replay_{l}.hfld"), out.replayed[l])


def test_bench_writes_csv(tmp_path):
    r = run("bench", "--grid", "32", "--n-list", "0,50", "--l-list", "1", "--out", str(tmp_path / "b.csv"))
    assert r.returncode == 0, r.stderr
    lines = (tmp_path / "b.csv").read_text().strip().splitlines()
    assert lines[0] == "n,l,raster_seconds,record_seconds,total_seconds"
    assert [ln.split(",")[:2] for ln in lines[1:]] == [["0", "1"], ["50", "1"]]
    assert all(float(ln.split(",")[4]) > 0 for ln in lines[1:])


def read_gray_png(path):
    """Minimal PNG reader for the grayscale 8 / 16-bit, filter-0 files `holo` writes."""
    import struct
    import zlib

    data = open(path, "rb").read()
    assert data[:8] == b"\x89PNG\r\n\x1a\n"
    pos, idat, w = 8, b"", None
    while pos < len(data):
        n = struct.unpack(">I", data[pos:pos + 4])[0]
        typ, body = data[pos + 4:pos + 8], data[pos + 8:pos + 8 + n]
        assert zlib.crc32(typ + body) == struct.unpack(">I", data[pos + 8 + n:pos + 12 + n])[0]
        if typ == b"IHDR":
            w, h, depth, color = struct.unpack(">IIBB", body[:10])
            assert color == 0
        elif typ == b"IDAT":
            idat += body
        pos += 12 + n
    raw = zlib.decompress(idat)
    bpp = depth // 8
    rows = [raw[y * (w * bpp + 1):(y + 1) * (w * bpp + 1)] for y in range(h)]
    assert all(r[0] == 0 for r in rows)
    a = np.frombuffer(b"".join(r[1:] for r in rows), dtype=">u2" if depth == 16 else "u1").reshape(h, w)
    return a.astype(np.int64), depth


def test_phase_only_emits_quantized_phase_planes(tmp_path, gpu_ctx):
    """test_cli.cpp:220-245: single-channel hologram, 5 iterations, 10-bit phase PNG."""
    rng = np.random.default_rng(4)
    P = rng.uniform(0.2, 1.0, (1, 32, 32)) * np.exp(1j * rng.uniform(0.0, 2 * np.pi, (1, 32, 32)))
    write_field(tmp_path / "holo.hfld", P)
    r = run("phase-only", "--in", str(tmp_path / "holo.hfld"), "--out", str(tmp_path / "phase.png"), "--iters", "5",
            "--bits", "10", "--wavelength", "532e-9")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["final_loss"] <= rep["initial_loss"]
    assert rep["files"] == [str(tmp_path / "phase.png")]  # one channel keeps the base name
    codes, depth = read_gray_png(tmp_path / "phase.png")
    assert codes.shape == (32, 32) and depth == 16
    phase = (codes >> 6) * (2 * np.pi / 1024)  # read_phase_png (png_io.cpp:189-200)
    assert np.all((phase >= 0.0) & (phase < 2 * np.pi))
    # the quantised planes are the conversion's own phases: same GPU conversion in process
    cfg = WaveConfig(nx=32, ny=32, wavelengths=(532e-9,), num_planes=2)
    res = api.convert_phase_only(P, cfg, 5, ctx=gpu_ctx)
    want = np.round(np.mod(res.hologram.phase[0], 2 * np.pi) / (2 * np.pi / 1024)).astype(np.int64) % 1024
    assert np.array_equal(codes >> 6, want)
    # three channels: _r / _g / _b files; bad bit depth: usage error, exit 2
    P3 = np.concatenate([P, P, P])
    write_field(tmp_path / "h3.hfld", P3)
    r = run("phase-only", "--in", str(tmp_path / "h3.hfld"), "--out", str(tmp_path / "p.png"), "--iters", "2")
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout)["files"] == [str(tmp_path / f"p_{c}.png") for c in "rgb"]
    assert read_gray_png(tmp_path / "p_g.png")[1] == 8
    bad = run("phase-only", "--in", str(tmp_path / "holo.hfld"), "--out", str(tmp_path / "x.png"), "--bits", "12")
    assert bad.returncode == 2 and json.loads(bad.stderr)["error"]["kind"] == "usage"
