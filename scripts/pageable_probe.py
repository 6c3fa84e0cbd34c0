#!/usr/bin/env python
"""Host-operand call cost with pageable vs pinned host memory (the reference's run_kernel
passes pageable numpy buffers)."""
import ctypes, sys, time
from pathlib import Path
import numpy as np
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native
lib = _native.load()
torch.cuda.set_device(0)
n = 16384
P = lambda t: ctypes.c_void_p(t.data_ptr())
import itertools
cases = [("pinned", 1, 0, 1), ("pageable", 0, 0, 1)] + [("pageable", 1, t, nt) for nt in (0, 1)
                                                         for t in (1, 2, 4, 8, 12, 16)]
for kind, bounce, threads, nt in cases:
    _native.set_tuning(host_bounce=bounce, host_threads=threads, host_nt=nt)
    mk = (lambda *s: torch.empty(*s, dtype=torch.float64, pin_memory=True)) if kind == "pinned" \
        else (lambda *s: torch.empty(*s, dtype=torch.float64))
    A = mk(n * n); A.uniform_(-1, 1)
    B = mk(n * n)
    v = [mk(n).uniform_(-1, 1) for _ in range(7)]
    o = [mk(n) for _ in range(3)]
    for name, fn, nbytes in (
        ("bicgk", lambda: lib.bicgk(P(A), P(v[0]), P(v[1]), P(o[0]), P(o[1]), n, n), 8.0 * n * n),
        ("gemver", lambda: lib.gemver(P(A), P(v[0]), P(v[1]), P(v[2]), P(v[3]), 0.5, 0.25, P(v[4]), P(v[5]),
                                      P(B), P(o[0]), P(o[1]), n, n), 16.0 * n * n)):
        fn(); _native.check()
        t0 = time.perf_counter()
        for _ in range(3):
            fn(); _native.check()
        dt = (time.perf_counter() - t0) / 3
        print(f"{kind:9s} bounce={bounce} threads={threads:2d} nt={nt} {name:7s} n={n}: {dt*1e3:8.1f} ms  PCIe payload {nbytes/dt/1e9:6.1f} GB/s", flush=True)
