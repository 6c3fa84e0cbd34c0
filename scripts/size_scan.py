#!/usr/bin/env python
"""GB/s of every hot-path sequence as a function of n (device-resident, CUDA events)."""
import ctypes
import json
import statistics
import sys
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native  # noqa: E402
from paper_1205_1098_b200.sharded import GpuShardOps  # noqa: E402

torch.cuda.set_device(0)
lib = _native.load()
ops = GpuShardOps()
rows = []
SIZES = tuple(int(a) for a in sys.argv[1:]) or (512, 1024, 2048, 4096, 8192, 16384)
for n in SIZES:
    A = torch.rand(n, n, dtype=torch.float64, device="cuda")
    B = torch.rand(n, n, dtype=torch.float64, device="cuda")
    v = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(8)]
    o = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
    big = torch.rand(4, min(n * n, 1 << 27), dtype=torch.float64, device="cuda")
    beta = torch.empty(1, dtype=torch.float64, device="cuda")
    calls = {
        "axpydot": (lambda: ops.axpydot(big[0], big[1], big[2], 0.3, big[3], beta), 32.0 * big.shape[1]),
        "bicgk": (lambda: ops.bicgk(A, v[0], v[1], o[0], o[1]), 8.0 * n * n),
        "atax": (lambda: ops.atax(A, v[0], o[0]), 8.0 * n * n),
        "gesummv": (lambda: ops.gesummv(0.5, 0.25, A, B, v[0], o[0]), 16.0 * n * n),
        "gemver": (lambda: ops.gemver(A, v[0], v[1], v[2], v[3], 0.5, 0.25, v[4], v[5], B, o[0], o[1]),
                   24.0 * n * n),
    }
    for name, (fn, nbytes) in calls.items():
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        evs = []
        for _ in range(30):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        us = statistics.median(a.elapsed_time(b) for a, b in evs) * 1e3
        # back-to-back (no events in between): amortised time per call
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            fn()
        b.record()
        torch.cuda.synchronize()
        us_b2b = a.elapsed_time(b) * 1e3 / 50
        rows.append({"kernel": name, "n": n, "us": us, "us_b2b": us_b2b, "gbs": nbytes / us / 1e3,
                     "gbs_b2b": nbytes / us_b2b / 1e3})
        print(f"n={n:6d} {name:8s} {us:9.1f} us  {nbytes / us / 1e3:7.0f} GB/s   "
              f"back-to-back {us_b2b:9.1f} us {nbytes / us_b2b / 1e3:7.0f} GB/s", flush=True)
Path(REPO / "gpurun_out").mkdir(exist_ok=True)
(REPO / "gpurun_out" / "size_scan.json").write_text(json.dumps(rows, indent=1))
