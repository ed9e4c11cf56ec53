"""Benchmark: hologram frames/sec of the forward render (BASELINE.json metric).

One step = one frame of holo::pipeline_forward (proj/src/pipeline.cpp:20-29):
raster -> forward recording -> inverse propagation -> intensities, for the
headline workload C3 (1M complex Gaussians, 1920x1080, 8 planes, RGB) on
synthetic data (scenes.py).  Outputs produced every step: the hologram
(complex64 [C,H,W]) and the L x C focal-stack intensities (float32).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

N > 1 runs under torchrun, one rank per GPU: planes are sharded across ranks and
the partial spectra are summed by one NCCL all-reduce per frame.
Rank 0 prints one JSON line.  ``--impl reference`` times the reference's own
C++ pipeline_forward (oracle/_ref, compiled from /root/reference/proj/src) on the
host cores, rank 0 only.
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


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ algorithmic bytes

def stage_bytes(N, L, C, P, E, planes_local, sharded, has_holo):
    """Algorithmic HBM bytes per frame and per stage.

    f = one C-channel complex64 field (C P 8 bytes); Lr = planes owned by this GPU;
    O = outputs of the inverse passes (the hologram on rank 0, plus the Lr planes)."""
    Lr = planes_local
    f = C * P * 8
    O = Lr + (1 if has_holo else 0)
    return {
        # f64 scene read + 64-B compositing record + 33 B of binning metadata per Gaussian
        "preprocess": N * (8 * (17 + L) + 64 + 33),
        # rect/count/plane re-read twice, bucket atomics, 4-B gidx entries written,
        # then sorted with their 8-B depth keys gathered
        "binning": N * 2 * 24 + E * (4 + 4 + 8),
        # sorted gidx list + 64-B record gather per entry, layers written once
        "composite": E * (4 + 64) + Lr * f,
        "fft_pass1": 2 * Lr * f,                                   # column FFT, in place
        "fft_pass2": Lr * f + (f if sharded else O * f),           # rows: read planes, write S or outputs
        "fft_pass3": f + O * f,                                    # rows from S (sharded only)
        "fft_pass4": O * f + (f if has_holo else 0) + Lr * C * P * 4,  # column IFFT + hologram / intensity
    }


STAGE_KERNEL = {"preprocess": "k_preprocess", "composite": "k_composite", "fft_pass1": "k_col_fwd",
                "fft_pass2": "k_row_fused", "fft_pass3": "k_row_fused", "fft_pass4": "k_col_inv_epi"}


def ncu_metric(stage, metric):
    """One column of the newest forward-frame ncu summary for the stage's kernel."""
    import csv
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r[0-9][0-9]_kernels.csv")))
    prefix = STAGE_KERNEL.get(stage)
    if not files or not prefix:
        return None
    for row in csv.DictReader(open(files[-1])):
        if row["kernel"].startswith(prefix) and row.get(metric):
            return float(row[metric])
    return None


def ncu_traffic(stage):
    """dram read + write bytes per launch of the stage's kernel from the newest
    committed forward-frame ncu --set full summary (profiles/rNN_kernels.csv), or None."""
    import csv
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r[0-9][0-9]_kernels.csv")))
    prefix = STAGE_KERNEL.get(stage)
    if not files or not prefix:
        return None
    for row in csv.DictReader(open(files[-1])):
        if row["kernel"].startswith(prefix):
            return float(row["dram__bytes_read.sum"]) + float(row["dram__bytes_write.sum"])
    return None


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
    cam = c.cameras()[0]
    scene = synthetic_scene(c.n, wave, c.seed)
    kind = "reference" if Oracle.available("ref") else "port"
    ora = Oracle("ref" if kind == "reference" else "restate")

    def frame():
        r = ora.pipeline_forward(scene, cam, wave, raster=False, replayed=False)
        return float(np.sum(r.stage_seconds)), r.stage_seconds

    return kind, frame


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
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
        "config": {"workload": f"{args.config}: reference pipeline_forward on host cores", "omp_threads": cores,
                   "steps_requested": args.steps, "warmup_requested": args.warmup},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": kind,
                         "sample": f"{steps} full {args.config} frames (steps capped to a {budget:.0f} s budget)"},
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=150.0)
    ap.add_argument("--inflight", type=int, default=2, help="frames in flight (contexts / streams) at N=1")
    ap.add_argument("--e2e-inflight", type=int, default=1, help="frames in flight in the end-to-end run at N=1")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2506_08350_b200 import _lib as L
    from paper_2506_08350_b200.api import Context
    from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    c = CONFIGS[args.config]
    wave = c.wave()
    cam = c.cameras()[0]
    Lp, Cn, H, W = wave.num_planes, wave.channels(), wave.ny, wave.nx
    P = H * W
    if Lp % world:
        raise SystemExit(f"{Lp} planes do not split over {world} ranks")
    pb, pe = rank * Lp // world, (rank + 1) * Lp // world
    scene = synthetic_scene(c.n, wave, c.seed)
    if world > 1:
        # hard plane assignment: each rank holds only its planes' Gaussians
        # (sharding.plane_subset; the rendered layers are unchanged)
        from paper_2506_08350_b200.sharding import plane_subset

        scene = plane_subset(scene, pb, pe)

    ctx = Context(local)
    ctx.upload_scene(scene)
    outs = L.OUT_INTENSITY | (L.OUT_HOLOGRAM if rank == 0 else 0)
    spec = torch.empty((Cn, H, W, 2), dtype=torch.float32, device=f"cuda:{local}") if world > 1 else None

    def frame():
        if world == 1:
            ctx.render(cam, wave, None, None, outputs=outs)
        else:
            ctx.render_begin(cam, wave, None, None, pb, pe, spec.data_ptr(), 0)
            dist.all_reduce(spec)
            ctx.render_end(wave, None, pb, pe, spec.data_ptr(), outs)

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
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            frame()
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ctx.frame_status()  # raises if any timed frame overflowed or failed validation
        launches = ctx.launch_count() - launches0
        ms = ev0.elapsed_time(ev1)
        t = torch.tensor([ms], device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_serial = float(t.item()) / args.steps

        # frames in flight on separate contexts / streams (1 GPU): the next frame's
        # raster overlaps the previous frame's tail kernels
        ms_pipe = None
        if world == 1 and args.inflight > 1:
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
    sb = stage_bytes(scene.size(), Lp, Cn, P, E, pe - pb, world > 1, rank == 0)
    stages = {}
    for name in STAGE_NAMES:
        tot_ms, calls = st[name]
        if calls == 0:
            continue
        avg = tot_ms / calls
        stages[name] = {"ms": avg, "bytes": sb[name], "GBps": sb[name] / (avg * 1e-3) / 1e9}
    dom = max(stages, key=lambda k: stages[k]["ms"])
    d = stages[dom]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": d["GBps"], "peak": hbm_peak, "unit": "GB/s",
                "frac": d["GBps"] / hbm_peak, "traffic": ncu_traffic(dom), "traffic_source": "profiles (ncu --set full, per launch)", "peak_kind": peak_kind,
                "frame_bytes": sum(sb.values()), "frame_frac": sum(sb.values()) / (ms_per_step * 1e-3) / 1e9 /
                (hbm_peak * world)}
    if dom == "composite":
        # compositing is FP32 / MUFU issue-bound, not HBM-bound: its
        # roofline is instruction issue; report the measured issue utilisation too
        ia = ncu_metric(dom, "smsp__issue_active.avg.pct_of_peak_sustained_active")
        roofline["compute"] = {"bound": "fp32/mufu issue", "issue_active": ia / 100.0 if ia is not None else None,
                               "source": "profiles (ncu --set full)"}

    # ---------------- end to end through the public API: pinned host scene in, results out
    # Every frame uploads the scene from pinned host memory and reads the hologram
    # and intensities back.  At N = 1 the frames rotate over `inflight` contexts on
    # their own streams, so one frame's upload, another's compute and a third's
    # download overlap on the two copy engines; at N > 1 each rank runs its shard
    # frame by frame.
    e2e = None
    if rank == 0 or world > 1:
        arrays = [np.ascontiguousarray(a, dtype=np.float64) for a in
                  (scene.positions, scene.rotations, scene.log_scales, scene.amplitudes, scene.opacity_logits,
                   scene.phases, scene.plane_logits)]
        pinned = [torch.from_numpy(a).pin_memory() for a in arrays]
        ptrs = [p.data_ptr() for p in pinned]
        h2d = sum(a.nbytes for a in arrays)
        n_e2e = max(20, min(args.steps, 60))
        nctx = max(1, args.e2e_inflight) if world == 1 else 1
        ectxs = [Context(local, use_torch_stream=False) for _ in range(nctx)] if world == 1 else [ctx]
        bufs = []
        for cx_ in ectxs:
            holo_h = torch.empty(Cn * P * 2, dtype=torch.float32).pin_memory() if rank == 0 else None
            int_h = torch.empty((pe - pb) * Cn * P, dtype=torch.float32).pin_memory()
            bufs.append((holo_h, int_h))
        d2h = bufs[0][1].numel() * 4 + (bufs[0][0].numel() * 4 if rank == 0 else 0)

        def e2e_step(i):
            cx_ = ectxs[i % len(ectxs)]
            holo_h, int_h = bufs[i % len(ectxs)]
            cx_.upload_scene_pointers(scene.size(), Lp, ptrs, device=False)
            if world == 1:
                cx_.render(cam, wave, None, None, outputs=outs)
            else:
                frame()
            if holo_h is not None:
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
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(n_e2e):
            e2e_step(i)
        for cx_ in ectxs:
            cx_.synchronize()
        torch.cuda.synchronize()
        el = torch.tensor([time.perf_counter() - t0], device=f"cuda:{local}")
        for cx_ in ectxs:
            cx_.frame_status()
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        e2e = {"value": n_e2e / float(el.item()), "unit": "frames/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": n_e2e, "frames_in_flight": len(ectxs)}
        if world == 1:
            for cx_ in ectxs:
                cx_.close()

    # ---------------- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            kind, ref_frame = reference_frame_seconds(args.config)
            tsec, split = ref_frame()
            cpu = {"value": 1.0 / tsec, "unit": "frames/s", "cores": os.cpu_count(), "kind": kind,
                   "sample": f"1 full {args.config} frame of pipeline_forward (raster {split[0]:.2f}s, record "
                             f"{split[1]:.2f}s, replay {split[2]:.2f}s, intensity {split[3]:.2f}s)"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "frames/s", "cores": os.cpu_count(), "kind": "unavailable",
                   "sample": f"oracle not runnable here: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp32 (f64 projection/keys)", "data": "synthetic",
            "config": {"workload": f"{args.config}: {c.n} Gaussians, {W}x{H}, {Lp} planes, {Cn} channels",
                       "parallelism": "planes sharded, NCCL all-reduce of the spectrum" if world > 1 else "1 GPU",
                       "entries": E, "l2": "per-frame working set (layers 398 MB, scene 200 MB) > 126 MB L2"},
            "latency_ms": ms_serial, "frames_in_flight": args.inflight if (ms_pipe is not None and ms_pipe < ms_serial) else 1,
            "ms_per_step_inflight": ms_pipe,
            "roofline": roofline, "stages": stages, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
