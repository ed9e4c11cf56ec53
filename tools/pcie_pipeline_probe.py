"""Emulated upload -> compute -> download pipeline with torch streams and events:
per-frame timeline of the copy-in, compute and copy-out streams."""
import torch

U, D = 200_000_000, 248_832_000
hin = [torch.empty(U, dtype=torch.uint8).pin_memory() for _ in range(2)]
hout = [torch.empty(D, dtype=torch.uint8).pin_memory() for _ in range(2)]
din = [torch.empty(U, dtype=torch.uint8, device="cuda") for _ in range(2)]
dout = [torch.empty(D, dtype=torch.uint8, device="cuda") for _ in range(2)]
work = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
cin, comp, cout = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
N = 12
ev = {k: [torch.cuda.Event(enable_timing=True) for _ in range(N)] for k in
      ("up0", "up1", "c0", "c1", "d0", "d1")}
free = [torch.cuda.Event() for _ in range(2)]
outfree = [torch.cuda.Event() for _ in range(2)]
base = torch.cuda.Event(enable_timing=True)


def compute(k):
    for _ in range(3):  # ~1.6 ms of HBM-heavy work
        work.mul_(1.0000001)


def run(double_out):
    torch.cuda.synchronize()
    base.record()
    for s in (cin, comp, cout):
        s.wait_event(base)
    for i in range(N):
        k = i & 1
        with torch.cuda.stream(cin):
            cin.wait_event(free[k])
            ev["up0"][i].record(cin)
            din[k].copy_(hin[k], non_blocking=True)
            ev["up1"][i].record(cin)
        with torch.cuda.stream(comp):
            comp.wait_event(ev["up1"][i])
            ev["c0"][i].record(comp)
            compute(k)
            free[k].record(comp)
            ko = k if double_out else 0
            comp.wait_event(outfree[ko])
            dout[ko].fill_(1)
            ev["c1"][i].record(comp)
        with torch.cuda.stream(cout):
            cout.wait_event(ev["c1"][i])
            ev["d0"][i].record(cout)
            hout[k].copy_(dout[ko], non_blocking=True)
            ev["d1"][i].record(cout)
            outfree[ko].record(cout)
    torch.cuda.synchronize()
    t = lambda e: base.elapsed_time(e)
    for i in range(N):
        print(f"  frame {i:2d}: up {t(ev['up0'][i]):7.2f}-{t(ev['up1'][i]):7.2f}  compute {t(ev['c0'][i]):7.2f}-"
              f"{t(ev['c1'][i]):7.2f}  down {t(ev['d0'][i]):7.2f}-{t(ev['d1'][i]):7.2f}")
    print(f"  period {(t(ev['d1'][N - 1]) - t(ev['d1'][N - 5])) / 4:.2f} ms/frame")


for dbl in (False, True):
    print("double-buffered outputs" if dbl else "single output buffer")
    run(dbl)
