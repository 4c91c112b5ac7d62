#!/usr/bin/env python3
"""PCIe ceiling probe: pinned H2D, D2H, and both concurrently (1 GiB chunks)."""
import json
import time

import torch

N = 8 << 30
h_src = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h_dst = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(N, dtype=torch.uint8, device="cuda")
d_b = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


for f in (h2d, d2h, both):
    timed(f)
out = {"h2d_GBps": N / timed(h2d) / 1e9, "d2h_GBps": N / timed(d2h) / 1e9}
t = timed(both)
out["concurrent_each_GBps"] = N / t / 1e9
out["concurrent_total_GBps"] = 2 * N / t / 1e9
print(json.dumps({k: round(v, 2) for k, v in out.items()}))
