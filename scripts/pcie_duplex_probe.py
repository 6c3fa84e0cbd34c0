#!/usr/bin/env python
"""Raw PCIe rates with pinned memory: one direction at a time, both at once, and both at once with
the copies cut into panels (what the host-operand pipeline does)."""
import time
import torch

torch.cuda.set_device(0)
GiB = 1 << 30
n = 4 * GiB // 8
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
h_in.fill_(1.0); d_out.fill_(2.0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d(); d2h()


def panels(mib):
    step = mib * (1 << 20) // 8
    def run():
        for o in range(0, n, step):
            with torch.cuda.stream(s1):
                d_in[o:o + step].copy_(h_in[o:o + step], non_blocking=True)
            with torch.cuda.stream(s2):
                h_out[o:o + step].copy_(d_out[o:o + step], non_blocking=True)
    return run


t = timed(h2d); print(f"H2D alone   {4 / t:6.1f} GiB/s = {4 * GiB / t / 1e9:6.1f} GB/s")
t = timed(d2h); print(f"D2H alone   {4 / t:6.1f} GiB/s = {4 * GiB / t / 1e9:6.1f} GB/s")
t = timed(both); print(f"both at once: each {4 * GiB / t / 1e9:6.1f} GB/s  ({t * 1e3:.1f} ms for 4 GiB each way)")
for mib in (16, 64, 256):
    t = timed(panels(mib)); print(f"both, {mib:3d} MiB panels: each {4 * GiB / t / 1e9:6.1f} GB/s  ({t * 1e3:.1f} ms)")
