"""Benchmark: hologram frames/sec of the forward render (BASELINE.json metric).

One step = one batch of holo::pipeline_forward frames (proj/src/pipeline.cpp:20-29):
raster -> forward recording -> inverse propagation -> intensities, on synthetic
scenes (scenes.py).  Outputs produced every frame: the hologram (complex64
[C,H,W]) and the L x C focal-stack intensities (float32).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

Workloads (BASELINE.json configs; --config):
  C3 (default, the metric's config): 1M Gaussians, 1920x1080, 8 planes, RGB; one
     view per step; at N > 1 the planes are sharded (holo_group_render: per-channel
     spectrum sum over NCCL overlapped with the next channel's row pass).
  C4: 64 views of a 1M-Gaussian scene at 1024^2, 6 planes per step, views sharded.
  C5: 8 views of a 3M-Gaussian scene at 3840x2160, 16 planes per step, planes x
     views (plane split 2 from N = 2 on).
  C1, C2: the smaller configurations, one view per step.
value = frames (views) of the whole job per second.  N > 1 runs under torchrun,
one rank per GPU; rank 0 prints one JSON line.  ``--impl reference`` times the
reference's own C++ pipeline_forward (oracle/_ref, compiled from
/root/reference/proj/src) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hologram frames/sec (1M Gaussians, 1920×1080, 8 planes, RGB); HBM roofline %"
STAGE_NAMES = ("preprocess", "binning", "composite", "fft_pass1", "fft_pass2", "fft_pass3", "fft_pass4")
FFT_STAGES = ("fft_pass1", "fft_pass2", "fft_pass3", "fft_pass4")


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ algorithmic bytes

def survey_frame_bytes(N, L, C, P, E):
    """B_frame = C P 8 (6.5 L + 3) + 88 E + N (8 (17 + L) + 84): the algorithmic
    HBM bytes of one frame on one GPU."""
    return C * P * 8 * (6.5 * L + 3) + 88 * E + N * (8 * (17 + L) + 84)


def stage_bytes(N, L, C, P, E, Lr=None, holo_frac=1.0, sharded=False):
    """The same model split over the stages this rank runs (planes Lr of L; the
    fraction holo_frac of the hologram's channels formed here).  f = one
    C-channel complex64 field.  Single GPU: the stages sum to survey_frame_bytes."""
    Lr = L if Lr is None else Lr
    f = C * P * 8
    h = holo_frac
    b = {"preprocess": N * (8 * (17 + L) + 84),    # f64 scene + 48-B record + 36-B depth rank
         "binning": 36 * E,                        # keys + values written, sort read + write
         "composite": 52 * E + Lr * f,             # index + record per entry, layers written
         "fft_pass1": 2 * Lr * f}                  # column FFT in place
    if not sharded:
        b["fft_pass2"] = Lr * f + (Lr + h) * f     # rows: planes in, replays + hologram out
        b["fft_pass4"] = (Lr + h) * f + h * f + Lr * f / 2  # columns: hologram + intensities out
    else:
        b["fft_pass2"] = Lr * f + f                # rows: planes in, partial spectrum out
        b["fft_pass3"] = f + (Lr + h) * f          # rows: summed spectrum in, replays out
        b["fft_pass4"] = (Lr + h) * f + h * f + Lr * f / 2
    return b


STAGE_KERNEL = {"preprocess": "k_preprocess", "composite": "k_composite", "fft_pass1": "k_col_fwd",
                "fft_pass2": "k_row_fused", "fft_pass3": "k_row_fused", "fft_pass4": "k_col_inv_epi"}


def _newest_profile():
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r[0-9][0-9]_kernels.csv")))
    return files[-1] if files else None


PROFILED_CONFIG = "C3"  # the configuration the committed forward-frame ncu summaries capture
_CONFIG = {"name": "C3"}


def ncu_metric(stage, metric):
    """One column of the newest forward-frame ncu summary for the stage's kernel
    (C3 captures: None for the other configurations)."""
    import csv

    path, prefix = _newest_profile(), STAGE_KERNEL.get(stage)
    if not path or not prefix or _CONFIG["name"] != PROFILED_CONFIG:
        return None
    for row in csv.DictReader(open(path)):
        if row["kernel"].startswith(prefix) and row.get(metric):
            return float(row[metric])
    return None


def ncu_traffic(stage):
    """dram read + write bytes per launch of the stage's kernel from the newest
    committed forward-frame ncu --set full summary (profiles/rNN_kernels.csv), or None."""
    r, w = ncu_metric(stage, "dram__bytes_read.sum"), ncu_metric(stage, "dram__bytes_write.sum")
    return None if r is None or w is None else r + w


# ------------------------------------------------------------------ clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        rows = [r for r in self.rows if num(r[0]) is not None]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        busy = [r for r in rows if (num(r[7]) or 0) > 0] or rows
        names = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
        reasons = sorted({n for r in busy for n, v in zip(names, r[3:7]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(num(r[0]) for r in busy), "sm_max_mhz": num(busy[0][1]),
                "power_w_max": max((num(r[2]) or 0) for r in busy), "reasons": reasons, "samples": len(busy)}


# ------------------------------------------------------------------ reference arm

def reference_frame_seconds(cfgname: str):
    from oracle.oracle import Oracle
    from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene

    c = CONFIGS[cfgname]
    wave = c.wave()
    cams = c.cameras()
    scene = synthetic_scene(c.n, wave, c.seed)
    kind = "reference" if Oracle.available("ref") else "port"
    ora = Oracle("ref" if kind == "reference" else "restate")
    state = {"k": 0}

    def frame():
        cam = cams[state["k"] % len(cams)]
        state["k"] += 1
        r = ora.pipeline_forward(scene, cam, wave, raster=False, replayed=False)
        return float(np.sum(r.stage_seconds)), r.stage_seconds

    return kind, frame


def fft_calibration():
    """The reference arm's FFT is the oracle's f64 shim over oracle/fft64.c (FFTW3
    is absent here): one 1920x1080 complex128 2-D FFT with it against numpy's
    pocketfft, both single-threaded on this host."""
    try:
        from oracle.oracle import Oracle

        rng = np.random.default_rng(0)
        x = rng.standard_normal((1, 1080, 1920)) + 1j * rng.standard_normal((1, 1080, 1920))
        ora = Oracle("restate")
        ora.fft2(x)
        t0 = time.perf_counter()
        ora.fft2(x)
        shim = time.perf_counter() - t0
        np.fft.fft2(x[0])
        t0 = time.perf_counter()
        np.fft.fft2(x[0])
        pocket = time.perf_counter() - t0
        return {"shim_fft_ms": 1e3 * shim, "pocketfft_ms": 1e3 * pocket, "shim_over_pocketfft": shim / pocket,
                "what": "one 1920x1080 complex128 FFT2, single thread: the reference arm's FFTW stand-in "
                        "(oracle/fft64.c) vs numpy pocketfft; the CPU baseline's propagation is this much slower "
                        "than with a pocketfft-class FFT"}
    except Exception as e:  # noqa: BLE001
        return {"error": repr(e)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # rank 0 alone runs the reference, on every host core: torchrun's default
    # OMP_NUM_THREADS=1 per process would leave its OpenMP loops single-threaded
    # (set before the reference library -- and its OpenMP runtime -- is loaded)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())
    kind, frame = reference_frame_seconds(args.config)
    cores = os.cpu_count()
    budget = args.ref_budget_s
    t_first, _ = frame()  # warm-up (page faults, OpenMP pool)
    steps = max(1, min(args.steps, int(budget / max(t_first, 1e-3))))
    times = []
    for _ in range(steps):
        t, _ = frame()
        times.append(t)
    total = float(np.sum(times))
    value = steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": 1, "ms_per_step": 1e3 * total / steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: reference pipeline_forward on host cores, one frame per step",
                   "omp_threads": cores, "steps_requested": args.steps, "warmup_requested": args.warmup},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": kind,
                         "sample": f"{steps} full {args.config} frames (steps capped to a {budget:.0f} s budget)",
                         "fft_calibration": fft_calibration()},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--plane-split", type=int, default=0, help="ranks per plane group (0: the config's policy)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dropin", action="store_true", help="skip the C++ drop-in API leg (e2e_dropin)")
    ap.add_argument("--ref-budget-s", type=float, default=150.0)
    ap.add_argument("--inflight", type=int, default=3, help="frames in flight (contexts / lanes) per GPU")
    ap.add_argument("--e2e-inflight", type=int, default=1, help="frames in flight in the end-to-end run at N=1")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.impl == "reference":
        run_reference(args)
        return

    # keep stdout to the one JSON line (NCCL prints a version banner at its first
    # communicator otherwise)
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    import torch
    import torch.distributed as dist

    from paper_2506_08350_b200.scenes import CONFIGS

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HOLO_BENCH_ONE_GPU=1 (dry runs of the N > 1 path on a one-GPU box): every rank
    # on cuda:0, torch.distributed over gloo and the group's spectrum sums through
    # gloo (NCCL refuses two ranks on one device); timings are then meaningless
    one_gpu = os.environ.get("HOLO_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    c = CONFIGS[args.config]
    _CONFIG["name"] = args.config
    if c.views == 1 and world == 1:
        res = run_single(args, c, local)
    else:
        res = run_group(args, c, world, rank, local)
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(args.config)
        res["cpu_baseline"] = cpu
        if world == 1 and c.views == 1 and not args.no_dropin:
            res["e2e_dropin"] = dropin_leg(c)
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


def dropin_leg(c):
    """holo::pipeline_forward through the C++ drop-in (libholo.so), timed by
    paper_2506_08350_b200/lib/dropin_bench with steady_clock as the reference times
    its own API (holo_main.cpp:507-514): scene in from host memory, the whole
    PipelineForward (f64 raster layers and lists, hologram, replayed fields,
    intensities) back in host memory, every call."""
    exe = os.path.join(ROOT, "paper_2506_08350_b200", "lib", "dropin_bench")
    if not os.path.exists(exe):
        return {"unavailable": "dropin_bench not built"}
    try:
        import tempfile

        from paper_2506_08350_b200.scenes import synthetic_scene, write_scene

        wave = c.wave()
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "scene.holoscene")
            write_scene(path, synthetic_scene(c.n, wave, c.seed))
            cmd = [exe, path, "--nx", str(wave.nx), "--ny", str(wave.ny), "--planes", str(wave.num_planes),
                   "--wavelengths", ",".join(repr(x) for x in wave.wavelengths), "--frames", "5", "--warmup", "1"]
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        if out.returncode != 0:
            return {"unavailable": out.stderr.strip()[-300:]}
        r = json.loads(out.stdout.strip().splitlines()[-1])
        r["unit"] = "frames/s"
        return r
    except Exception as e:  # noqa: BLE001
        return {"unavailable": repr(e)}


def cpu_baseline(cfgname):
    try:
        kind, ref_frame = reference_frame_seconds(cfgname)
        tsec, split = ref_frame()
        return {"value": 1.0 / tsec, "unit": "frames/s", "cores": os.cpu_count(), "kind": kind,
                "sample": f"1 full {cfgname} frame of pipeline_forward (raster {split[0]:.2f}s, record "
                          f"{split[1]:.2f}s, replay {split[2]:.2f}s, intensity {split[3]:.2f}s)",
                "fft_calibration": fft_calibration()}
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": "frames/s", "cores": os.cpu_count(), "kind": "unavailable",
                "sample": f"oracle not runnable here: {e}"}


def roofline_block(stages, frame_bytes_1gpu, frames_per_s, world, hbm_peak, peak_kind, design_note):
    """The dominant stage's roofline (algorithmic bytes per frame / its time per
    frame), every FFT pass's fraction, and the whole-frame fraction: single-GPU
    B_frame x frames/s / (world x peak)."""
    dom = max(stages, key=lambda k: stages[k]["ms"])
    d = stages[dom]
    rl = {"bound": "hbm", "kernel": dom, "achieved": d["GBps"], "peak": hbm_peak, "unit": "GB/s",
          "frac": d["GBps"] / hbm_peak, "traffic": ncu_traffic(dom),
          "traffic_source": "profiles (ncu --set full, dram bytes per launch)", "peak_kind": peak_kind,
          "bytes_model": "SURVEY.md 8(d) per-stage terms", "frame_bytes": frame_bytes_1gpu,
          "frame_frac": frame_bytes_1gpu * frames_per_s / 1e9 / (hbm_peak * world),
          "fft_frac": {k: stages[k]["GBps"] / hbm_peak for k in FFT_STAGES if k in stages}}
    fft_ms = sum(stages[k]["ms"] for k in FFT_STAGES if k in stages)
    fft_b = sum(stages[k]["bytes"] for k in FFT_STAGES if k in stages)
    if fft_ms > 0:
        rl["fft_frac"]["propagation"] = fft_b / (fft_ms * 1e-3) / 1e9 / hbm_peak
    if dom == "composite":
        # compositing is FP32 / MUFU issue-bound, not HBM-bound: its
        # roofline is instruction issue; report the measured issue utilisation too
        ia = ncu_metric(dom, "smsp__issue_active.avg.pct_of_peak_sustained_active")
        rl["compute"] = {"bound": "fp32/mufu issue", "issue_active": ia / 100.0 if ia is not None else None,
                         "source": "profiles (ncu --set full)"}
    rl["note"] = design_note
    return rl


def stage_table(st, frames, sb):
    out = {}
    for name in STAGE_NAMES:
        tot_ms, calls = st[name]
        if calls == 0 or name not in sb:
            continue
        ms = tot_ms / frames
        out[name] = {"ms": ms, "launches_per_frame": calls / frames, "bytes": sb[name],
                     "GBps": sb[name] / (ms * 1e-3) / 1e9}
    return out


def run_single(args, c, local):
    """One GPU, one view per step: holo_render on `inflight` contexts / streams."""
    import torch

    from paper_2506_08350_b200 import _lib as L
    from paper_2506_08350_b200.api import Context
    from paper_2506_08350_b200.scenes import synthetic_scene

    wave = c.wave()
    cam = c.cameras()[0]
    Lp, Cn, H, W = wave.num_planes, wave.channels(), wave.ny, wave.nx
    P = H * W
    scene = synthetic_scene(c.n, wave, c.seed)
    ctx = Context(local)
    ctx.upload_scene(scene)
    outs = L.OUT_INTENSITY | L.OUT_HOLOGRAM

    def frame():
        ctx.render(cam, wave, None, None, outputs=outs)

    for _ in range(args.warmup):
        frame()
    torch.cuda.synchronize()
    E = int(ctx.info.num_entries)
    # asynchronous frames from here on: no host round trip inside a frame; the
    # entry buffers keep the capacity the synchronous warm-up frames reserved
    ctx.set_async(True)
    for _ in range(2):
        frame()
    ctx.frame_status()

    # ---------------- timed region: device-resident inputs, CUDA events on the launch stream
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            frame()
        ev1.record(stream)
        torch.cuda.synchronize()
        ctx.frame_status()  # raises if any timed frame overflowed or failed validation
        launches = ctx.launch_count() - launches0
        ms_serial = ev0.elapsed_time(ev1) / args.steps

        # frames in flight on separate contexts / streams: the next frame's raster
        # overlaps the previous frame's tail kernels
        ms_pipe = None
        if args.inflight > 1:
            extra = []
            for _ in range(args.inflight - 1):
                cx_ = Context(local, use_torch_stream=False)
                cx_.upload_scene(scene)
                cx_.render(cam, wave, None, None, outputs=outs)
                cx_.set_async(True)
                extra.append(cx_)
            ctxs = [ctx] + extra
            streams = [stream] + [torch.cuda.ExternalStream(cx_.stream()) for cx_ in extra]
            evs = [torch.cuda.Event() for _ in extra]

            def pipelined(n):
                ev0.record(stream)
                for s_ in streams[1:]:
                    s_.wait_event(ev0)
                for i in range(n):
                    ctxs[i % len(ctxs)].render(cam, wave, None, None, outputs=outs)
                for s_, e_ in zip(streams[1:], evs):
                    e_.record(s_)
                    stream.wait_event(e_)
                ev1.record(stream)

            pipelined(2 * len(ctxs))
            torch.cuda.synchronize()
            l0 = sum(cx_.launch_count() for cx_ in ctxs)
            pipelined(args.steps)
            torch.cuda.synchronize()
            for cx_ in ctxs:
                cx_.frame_status()
            launches = sum(cx_.launch_count() for cx_ in ctxs) - l0
            ms_pipe = ev0.elapsed_time(ev1) / args.steps
            for cx_ in extra:
                cx_.close()
    ms_per_step = ms_serial if ms_pipe is None else min(ms_serial, ms_pipe)
    fps = 1e3 / ms_per_step

    # ---------------- per-stage CUDA-event times (separate pass, same stream)
    ctx.reset_timing()
    ctx.enable_timing(True)
    nstage = min(args.steps, 20)
    for _ in range(nstage):
        frame()
    st = ctx.stage_times()
    ctx.enable_timing(False)
    hbm_peak, peak_kind = load_peaks()
    sb = stage_bytes(scene.size(), Lp, Cn, P, E)
    stages = stage_table(st, nstage, sb)
    B = survey_frame_bytes(scene.size(), Lp, Cn, P, E)
    roofline = roofline_block(stages, B, fps, 1, hbm_peak, peak_kind,
                              "frame_bytes = SURVEY 8(d) B_frame with the measured E; stages sum to it")

    # ---------------- end to end through the public API: pinned host scene in, results out
    # Every frame uploads the scene from pinned host memory and reads the hologram
    # and intensities back.  The frames rotate over `e2e_inflight` contexts on their
    # own streams, so one frame's upload, another's compute and a third's download
    # overlap on the two copy engines.
    arrays = [np.ascontiguousarray(a, dtype=np.float64) for a in
              (scene.positions, scene.rotations, scene.log_scales, scene.amplitudes, scene.opacity_logits,
               scene.phases, scene.plane_logits)]
    pinned = [torch.from_numpy(a).pin_memory() for a in arrays]
    ptrs = [p.data_ptr() for p in pinned]
    h2d = sum(a.nbytes for a in arrays)
    n_e2e = max(20, min(args.steps, 60))
    ectxs = [Context(local, use_torch_stream=False) for _ in range(max(1, args.e2e_inflight))]
    bufs = [(torch.empty(Cn * P * 2, dtype=torch.float32).pin_memory(),
             torch.empty(Lp * Cn * P, dtype=torch.float32).pin_memory()) for _ in ectxs]
    d2h = (bufs[0][0].numel() + bufs[0][1].numel()) * 4

    def e2e_step(i):
        cx_ = ectxs[i % len(ectxs)]
        holo_h, int_h = bufs[i % len(ectxs)]
        cx_.upload_scene_pointers(scene.size(), Lp, ptrs, device=False)
        cx_.render(cam, wave, None, None, outputs=outs)
        cx_.download_into(L.BUF_HOLOGRAM, holo_h.data_ptr(), holo_h.numel() * 4, wait=False)
        cx_.download_into(L.BUF_INTENSITY, int_h.data_ptr(), int_h.numel() * 4, wait=False)

    for i in range(len(ectxs)):  # synchronous first frames size the buffers, then asynchronous
        e2e_step(i)
        ectxs[i].synchronize()
        ectxs[i].set_async(True)
    for i in range(len(ectxs)):
        e2e_step(i)
    for cx_ in ectxs:
        cx_.synchronize()
    t0 = time.perf_counter()
    for i in range(n_e2e):
        e2e_step(i)
    for cx_ in ectxs:
        cx_.synchronize()
    el = time.perf_counter() - t0
    for cx_ in ectxs:
        cx_.frame_status()
        cx_.close()
    e2e = {"value": n_e2e / el, "unit": "frames/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "steps": n_e2e, "frames_in_flight": len(ectxs), "api": "Context.render (holo_render) from pinned host"}

    return {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "fp32 (f64 projection/keys)", "data": "synthetic",
        "config": {"workload": f"{c.name}: {c.n} Gaussians, {W}x{H}, {Lp} planes, {Cn} channels, 1 view per step",
                   "parallelism": "1 GPU", "entries": E,
                   "l2": "per-frame working set (layers 398 MB, scene 200 MB at C3) > 126 MB L2"},
        "latency_ms": ms_serial,
        "frames_in_flight": args.inflight if (ms_pipe is not None and ms_pipe < ms_serial) else 1,
        "ms_per_step_inflight": ms_pipe, "roofline": roofline, "stages": stages, "e2e": e2e,
        "gpu_launches": launches, "clocks": clk.summary(),
    }


def run_group(args, c, world, rank, local):
    """N GPUs (one process each) or a multi-view batch: holo_group_render.  Planes
    (C3 at N > 1), views (C4) or planes x views (C5); a step renders the batch's
    views (this rank's share of them)."""
    import torch
    import torch.distributed as dist

    from paper_2506_08350_b200 import _lib as L
    from paper_2506_08350_b200.api import Context, Group
    from paper_2506_08350_b200.scenes import synthetic_scene

    wave = c.wave()
    cams = c.cameras()
    V = len(cams)
    Lp, Cn, H, W = wave.num_planes, wave.channels(), wave.ny, wave.nx
    P = H * W
    if args.plane_split:
        ps = args.plane_split
    elif c.shard == "views":
        ps = 1
    elif c.shard == "planes_views":
        ps = 2 if world % 2 == 0 else 1
    else:
        ps = world
    scene = synthetic_scene(c.n, wave, c.seed)
    ctx = Context(local)
    if world > 1:
        if os.environ.get("HOLO_BENCH_ONE_GPU") == "1":
            from paper_2506_08350_b200.api import gloo_allreduce
            from paper_2506_08350_b200.sharding import torch_plane_group

            g = Group(ctx, world, rank, ps, allreduce=gloo_allreduce(torch_plane_group(ps)))
        else:
            g = Group.from_torch(ctx, plane_split=ps)
    else:
        g = Group(ctx, plane_split=1)
    if args.inflight > 1:
        g.set_lanes(args.inflight)
    g.upload_scene(scene)
    m = g.mesh(Lp, V, Cn)
    np_ = m.plane_end - m.plane_begin
    nv = m.view_end - m.view_begin
    hc = bin(m.holo_channels).count("1")
    outs = L.OUT_INTENSITY | L.OUT_HOLOGRAM
    # every view of the rank's share lands in its own caller buffers
    vouts = {v: (torch.empty((Cn, H, W), dtype=torch.complex64, device=f"cuda:{local}"), None,
                 torch.empty((max(np_, 1), Cn, H, W), dtype=torch.float32, device=f"cuda:{local}"))
             for v in range(m.view_begin, m.view_end)}

    def step():
        return g.render(cams, wave, None, None, outs, 0, vouts)

    infos = step()  # synchronous: per-view entry counts, sizes the entry buffers
    g.synchronize()
    E_views = {v: int(infos[v].num_entries) for v in range(m.view_begin, m.view_end)}
    for _ in range(args.warmup - 1):
        step()
    g.synchronize()
    g.set_async(True)
    for _ in range(2 * max(1, args.inflight)):  # every lane's first asynchronous frame (buffer growth)
        step()
    g.synchronize()
    g.frame_status()

    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = g.launch_count()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        g.join(stream.cuda_stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        g.synchronize()
        if world > 1:
            dist.barrier()
        g.frame_status()
        launches = g.launch_count() - l0
        t = torch.tensor([ev0.elapsed_time(ev1)], device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_per_step = float(t.item()) / args.steps
    fps = V * 1e3 / ms_per_step  # frames (views) of the whole job per second

    # ---------------- per-stage times of this rank (one lane, synchronous frames)
    g.set_async(False)
    g.set_lanes(1)
    ctx.reset_timing()
    ctx.enable_timing(True)
    nstage = max(1, min(args.steps, 5))
    for _ in range(nstage):
        step()
    g.synchronize()
    st = ctx.stage_times()
    ctx.enable_timing(False)
    hbm_peak, peak_kind = load_peaks()
    frames = nstage * nv
    E_r = float(np.mean(list(E_views.values()))) if E_views else 0.0
    sharded = ps > 1
    from paper_2506_08350_b200.sharding import hard_planes

    hp = hard_planes(scene)
    n_local = int(np.count_nonzero((hp >= m.plane_begin) & (hp < m.plane_end))) if sharded else c.n
    sb = stage_bytes(n_local, Lp, Cn, P, E_r, Lr=np_, holo_frac=hc / Cn, sharded=sharded)
    stages = stage_table(st, frames, sb) if frames else {}
    # whole-job frame roofline: single-GPU B_frame per view, E summed over the plane group
    E_tot = torch.tensor([sum(E_views.values())], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(E_tot)
    E_view_full = float(E_tot.item()) / V  # every view's entries are split over its plane group
    B = survey_frame_bytes(c.n, Lp, Cn, P, E_view_full)
    roofline = roofline_block(stages, B, fps, world, hbm_peak, peak_kind,
                              "frame_frac = single-GPU B_frame (SURVEY 8(d), measured E) x frames/s / "
                              "(n_gpus x peak); stage figures are rank 0's share") if stages else None

    # ---------------- end to end: scene uploaded from pinned host, every view's outputs read back
    arrays = [np.ascontiguousarray(a, dtype=np.float64) for a in
              (scene.positions, scene.rotations, scene.log_scales, scene.amplitudes, scene.opacity_logits,
               scene.phases, scene.plane_logits)]
    pinned = [torch.from_numpy(a).pin_memory() for a in arrays]
    from paper_2506_08350_b200.holotypes import GaussianScene

    pscene = GaussianScene(num_planes=Lp)
    for name, t_ in zip(("positions", "rotations", "log_scales", "amplitudes", "opacity_logits", "phases",
                         "plane_logits"), pinned):
        setattr(pscene, name, t_.numpy())
    hbufs = {v: (torch.empty((Cn, H, W), dtype=torch.complex64).pin_memory(),
                 torch.empty((max(np_, 1), Cn, H, W), dtype=torch.float32).pin_memory()) for v in vouts}
    h2d = sum(a.nbytes for a in arrays)
    d2h = sum(hc * P * 8 + np_ * Cn * P * 4 for _ in vouts)
    n_e2e = max(3, min(args.steps, 10))

    def e2e_step():
        g.upload_scene(pscene)
        step()
        g.join(stream.cuda_stream)
        for v, (hh, ii) in hbufs.items():
            if hc:
                hh.copy_(vouts[v][0], non_blocking=True)
            if np_:
                ii.copy_(vouts[v][2], non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        e2e_step()
    torch.cuda.synchronize()
    g.synchronize()
    el = torch.tensor([time.perf_counter() - t0], device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    e2e = {"value": V * n_e2e / float(el.item()), "unit": "frames/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": n_e2e,
           "api": "Group.upload_scene + Group.render (holo_group_*) from pinned host, outputs to pinned host"}
    g.close()
    ctx.close()
    shard = {1: "views"}.get(ps, "planes" if ps == world else "planes x views")
    return {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong",  # the batch (1, 64 or 8 views) is fixed: total work fixed
        "vs_baseline": None, "dtype": "fp32 (f64 projection/keys)", "data": "synthetic",
        "config": {"workload": f"{c.name}: {c.n} Gaussians, {W}x{H}, {Lp} planes, {Cn} channels, "
                               f"{V} view(s) per step",
                   "parallelism": f"{shard}: plane split {ps} x {world // ps} view groups (holo_group_render, "
                                  f"NCCL spectrum sum per channel)" if world > 1 else
                                  f"1 GPU, {V} views per step, {args.inflight} lanes",
                   "entries_per_view": E_view_full, "views": V,
                   "l2": "per-frame working set > 126 MB L2"},
        "roofline": roofline, "stages": stages, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
        "frames_in_flight": args.inflight,
    }


if __name__ == "__main__":
    main()
