"""Pinned host <-> device copy bandwidth, alone and with both directions at once."""
import time

import torch

h2d_b, d2h_b = 200_000_000, 248_832_000
hin = torch.empty(h2d_b, dtype=torch.uint8).pin_memory()
hout = torch.empty(d2h_b, dtype=torch.uint8).pin_memory()
din = torch.empty(h2d_b, dtype=torch.uint8, device="cuda")
dout = torch.empty(d2h_b, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(kind, n=10):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        if kind in ("h2d", "both"):
            with torch.cuda.stream(s1):
                din.copy_(hin, non_blocking=True)
        if kind in ("d2h", "both"):
            with torch.cuda.stream(s2):
                hout.copy_(dout, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n


for k in ("h2d", "d2h", "both"):
    run(k, 2)
    dt = run(k)
    print(f"{k}: {dt * 1e3:.2f} ms/iter  h2d {h2d_b / dt / 1e9 if k != 'd2h' else 0:.1f} GB/s  "
          f"d2h {d2h_b / dt / 1e9 if k != 'h2d' else 0:.1f} GB/s")
