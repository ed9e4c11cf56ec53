"""Summarise ncu output into profiles/ (committed evidence).

    python tools/ncu_summary.py --round r01 --launches gpurun_out/launches_r1.csv \
        --report gpurun_out/prof_r1.ncu-rep

Writes profiles/<round>_launches.csv (kernel, count, total and mean device time,
share of the timed frames), profiles/<round>_kernels.csv (per profiled launch:
duration, DRAM read/write bytes, achieved DRAM GB/s, registers, occupancy, issue
activity and the top stall reasons) and profiles/<round>_summary.md.
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    m = re.search(r"(k_[A-Za-z0-9_]+)(<[^(]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    agg = collections.OrderedDict()
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui] if ui is not None else "nsecond"
        us = v / 1000.0 if unit.startswith("ns") or unit == "nsecond" else (v if unit.startswith("us") else v * 1000.0)
        k = short(r[ki])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += us
    return agg


RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "smsp__inst_executed.sum"]
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "wait", "not_selected", "mio_throttle",
          "math_pipe_throttle", "lg_throttle", "dispatch_stall", "no_instruction"]


def to_base(v, unit):
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
    return v * scale.get(unit, 1)


def kernels(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        rec = {"kernel": short(d[hdr.index("Kernel Name")])}
        for m in RAW:
            if m in hdr:
                i = hdr.index(m)
                rec[m] = to_base(d[i], units[i]) if units[i] else float(d[i].replace(",", ""))
        for s in STALLS:
            m = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if m in hdr:
                rec["stall_" + s] = float(d[hdr.index(m)].replace(",", ""))
        t = rec.get("gpu__time_duration.sum", 0)
        rec["dram_GBps"] = (rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)) / t / 1e9 if t else 0
        res.append(rec)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", required=True)
    ap.add_argument("--launches", required=True)
    ap.add_argument("--report", required=True)
    ap.add_argument("--frames", type=int, default=10, help="frames in the ncu'd run (warmup + steps + stage pass)")
    args = ap.parse_args()
    pdir = os.path.join(ROOT, "profiles")
    os.makedirs(pdir, exist_ok=True)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}

    agg = launches(args.launches)
    total = sum(v[1] for v in agg.values())
    with open(os.path.join(pdir, f"{args.round}_launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_us", "mean_us", "share"])
        for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            w.writerow([k, n, f"{us:.1f}", f"{us / n:.2f}", f"{us / total:.4f}"])

    ks = kernels(args.report)
    cols = ["kernel", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram_GBps",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"] + ["stall_" + s for s in STALLS]
    with open(os.path.join(pdir, f"{args.round}_kernels.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(cols)
        for r in ks:
            w.writerow([r.get(c, "") if isinstance(r.get(c, ""), str) else f"{r.get(c):.6g}" for c in cols])

    lines = [f"# ncu summary — round {args.round}", "",
             f"HBM peak (MEASURED_PEAKS.json, measured): {peaks['hbm_gbs']} GB/s.", "",
             "## Launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised)", "",
             "| kernel | launches | total µs | mean µs | share |", "|---|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {us:.0f} | {us / n:.1f} | {us / total:.1%} |")
    lines += ["", "## Full-set capture of one frame's kernels", "",
              "| kernel | µs | DRAM read MB | DRAM write MB | DRAM GB/s | % of peak | regs | warps active % | issue active % | top stalls |",
              "|---|---|---|---|---|---|---|---|---|---|"]
    for r in ks:
        st = sorted(((r.get("stall_" + s, 0), s) for s in STALLS), reverse=True)[:3]
        lines.append(
            f"| `{r['kernel']}` | {r['gpu__time_duration.sum'] * 1e6:.1f} | {r['dram__bytes_read.sum'] / 1e6:.1f} | "
            f"{r['dram__bytes_write.sum'] / 1e6:.1f} | {r['dram_GBps']:.0f} | {r['dram_GBps'] / peaks['hbm_gbs']:.0%} | "
            f"{r.get('launch__registers_per_thread', 0):.0f} | "
            f"{r.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.0f} | "
            f"{r.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.0f} | "
            + ", ".join(f"{s} {v:.2f}" for v, s in st) + " |")
    open(os.path.join(pdir, f"{args.round}_summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
