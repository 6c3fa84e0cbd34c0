#!/usr/bin/env python
"""GEMVER's two passes timed separately over matrix sizes (aligned and not):  gemver_passes_probe.py [n ...]"""
import ctypes, statistics, sys
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native

lib = _native.load()
P = lambda t: ctypes.c_void_p(t.data_ptr())
sizes = [int(a) for a in sys.argv[1:] if a.isdigit()] or [12288, 14000, 16384, 24576, 30000, 32768]
for n in sizes:
    A = torch.rand(n, n, dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    v = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(6)]
    col = torch.empty(n, dtype=torch.float64, device="cuda"); w = torch.empty(n, dtype=torch.float64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    calls = {
        "pass1 (A -> B, B'y)": (lambda: lib.bto_gemver_pass1_async(P(A), P(v[0]), P(v[1]), P(v[2]), P(v[3]), P(v[4]), P(B), P(col), n, n, st), 16.0),
        "pass2 (B x)": (lambda: lib.bto_gemver_pass2_async(P(B), P(v[5]), 0.5, P(w), n, n, st), 8.0),
    }
    for name, (fn, per) in calls.items():
        for _ in range(3):
            _native.check(fn())
        torch.cuda.synchronize()
        ev = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); ev.append((a, b))
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in ev)
        print(f"n={n:6d} {name:22s} {ms:8.4f} ms {per * n * n / ms / 1e6:7.0f} GB/s  {_native.launch_plan()}", flush=True)
    del A, B

if "--sweep" in sys.argv:
    import itertools
    for n in (24576, 30000):
        A = torch.rand(n, n, dtype=torch.float64, device="cuda")
        B = torch.empty_like(A)
        v = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(6)]
        col = torch.empty(n, dtype=torch.float64, device="cuda")
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        fn = lambda: lib.bto_gemver_pass1_async(P(A), P(v[0]), P(v[1]), P(v[2]), P(v[3]), P(v[4]), P(B), P(col), n, n, st)
        rows = []
        for R, V, g, mb in itertools.product((0, 8, 16, 32), (0, 1, 2), (0, 1, 2, 3, 4, 8), (0, 1, 2)):
            try:
                _native.set_tuning(mv_rows=R, mv_vec=V, grid_per_sm=g, mv_minb=mb)
                for _ in range(2):
                    _native.check(fn())
                torch.cuda.synchronize()
                ev = []
                for _ in range(7):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(); fn(); b.record(); ev.append((a, b))
                torch.cuda.synchronize()
                ms = statistics.median(a.elapsed_time(b) for a, b in ev)
                rows.append((16.0 * n * n / ms / 1e6, R, V, g, mb, _native.launch_plan()))
            except Exception as exc:
                pass
        rows.sort(reverse=True)
        for r in rows[:6] + [x for x in rows if x[1:5] == (0, 0, 0, 0)]:
            print(f"n={n} pass1 {r[0]:7.0f} GB/s  mv_rows={r[1]} mv_vec={r[2]} grid_per_sm={r[3]} mv_minb={r[4]}  {r[5]}", flush=True)
        _native.set_tuning(mv_rows=0, mv_vec=0, grid_per_sm=0, mv_minb=0)
        del A, B
