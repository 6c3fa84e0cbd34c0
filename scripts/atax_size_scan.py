#!/usr/bin/env python
"""ATAX GB/s over matrix sizes whose column count is not a power of two (the slice per CTA is then
not a whole number of 512-column iterations):  atax_size_scan.py [tag]"""
import statistics
import sys
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native  # noqa: E402
from paper_1205_1098_b200.sharded import GpuShardOps  # noqa: E402

torch.cuda.set_device(0)
_native.load()
ops = GpuShardOps()
shapes = [(8192, 8192), (10240, 10240), (12288, 12288), (16384, 16384), (20480, 20480), (24576, 24576),
          (28672, 28672), (32768, 32768), (30000, 30000), (20000, 18000), (50000, 6000), (16384, 2560),
          (65536, 1536), (12000, 40960)]
if len(sys.argv) > 1:          # atax_size_scan.py 4096x65536 2048x131072 ...
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for (m, n) in shapes:
    A = torch.rand(m, n, dtype=torch.float64, device="cuda")
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(5):
        ops.atax(A, x, y)
    torch.cuda.synchronize()
    evs = []
    for _ in range(30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); ops.atax(A, x, y); b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in evs)
    plan = _native.launch_plan() if hasattr(_native, "launch_plan") else ""
    ref = A.t() @ (A @ x)
    err = float((y - ref).abs().max() / ref.abs().max())
    print(f"{m:6d} x {n:6d}  {ms:8.4f} ms  {8.0 * m * n / ms / 1e6:7.0f} GB/s  err {err:.1e}  {plan}", flush=True)
    del A
