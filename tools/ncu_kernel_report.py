"""Per-kernel digest of an ncu report: headline metrics, stall reasons, and the
source lines / SASS opcodes with the most instructions and stall samples.

    python tools/ncu_kernel_report.py gpurun_out/prof.ncu-rep k_row_fused [--top 20]
"""
import argparse
import collections
import csv
import io
import subprocess


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def ncu(*args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=20)
    a = ap.parse_args()
    rows = list(csv.reader(io.StringIO(ncu(a.report, "--page", "raw", "--csv", "-k", f"regex:{a.kernel}"))))
    h = rows[0]
    want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "dram__bytes_read.sum", "dram__bytes_write.sum"]
    for r in rows[2:]:
        print(r[h.index("Kernel Name")][:100])
        for w in want:
            if w in h:
                print(f"   {w:55s} {r[h.index(w)]}")
        st = [(float(r[i] or 0), h[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled")
              and not h[i].endswith("not_issued")]
        tot = sum(s for s, _ in st) or 1
        print("   stalls:", ", ".join(f"{n.split('stalled_')[1]} {s / tot * 100:.0f}%" for s, n in sorted(st, reverse=True)[:8]))
    src = list(csv.reader(io.StringIO(ncu(a.report, "--page", "source", "--csv", "-k", f"regex:{a.kernel}",
                                          "--print-source=cuda,sass"))))
    hdr, fname, lines, ops = None, None, [], collections.Counter()
    opstall = collections.Counter()
    for r in src:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        d = dict(zip(hdr, r))
        if r[0] != "":
            lines.append((num(r[4]), num(r[7]), f"{fname}:{r[0]}", r[1][:90]))
        else:
            tok = r[3].split()
            if not tok:
                continue
            op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
            ops[op.split(".")[0]] += num(r[7])
            opstall[op.split(".")[0]] += num(r[4])
    ts = sum(x[0] for x in lines) or 1
    te = sum(x[1] for x in lines) or 1
    print(f"\n   top source lines (stall-sample %, instruction %), total inst {te:.0f}")
    for s, e, loc, text in sorted(lines, key=lambda x: -(x[0] / ts + x[1] / te))[:a.top]:
        print(f"   {s / ts * 100:5.1f} {e / te * 100:5.1f}  {loc:24s} {text}")
    to = sum(ops.values()) or 1
    print("\n   opcodes:", ", ".join(f"{k} {v / to * 100:.1f}%" for k, v in ops.most_common(16)))


if __name__ == "__main__":
    main()
