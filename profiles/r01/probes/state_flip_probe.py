#!/usr/bin/env python
"""Bench-suite kernels before / after streaming the most recently allocated device memory."""
import ctypes, sys
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from bench import Suite, SUITE, BENCH, bytes_min  # noqa: E402
from paper_1205_1098_b200 import _native  # noqa: E402
torch.cuda.set_device(0)
lib = _native.load()
suite = Suite(torch, 0, 1, SUITE)
def measure(label, steps=10):
    for _ in range(3):
        for k in SUITE: suite.launch(k)
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in SUITE] for _ in range(steps)]
    for s in range(steps):
        for i, k in enumerate(SUITE):
            ev[s][i][0].record(); suite.launch(k); ev[s][i][1].record()
    torch.cuda.synchronize()
    out = {}
    for i, k in enumerate(SUITE):
        ms = sorted(ev[s][i][0].elapsed_time(ev[s][i][1]) for s in range(steps))[steps // 2]
        out[k] = round(bytes_min(k, *BENCH[k]) / ms / 1e6)
    print(f"{label:40s} {out}", flush=True)
measure("as allocated")
mode = sys.argv[1] if len(sys.argv) > 1 else "axpydot"
n = 1 << 27
fresh = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(4)]
beta = torch.empty(1, dtype=torch.float64, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
measure("after allocating+filling 4 GiB more")
if mode == "axpydot":
    _native.check(lib.bto_axpydot_async(P(fresh[0]), P(fresh[1]), P(fresh[2]), 0.37, P(fresh[3]), P(beta), n, st))
elif mode == "sum":
    for f in fresh: torch.sum(f)
elif mode == "sumlast":
    torch.sum(fresh[3])
torch.cuda.synchronize()
measure(f"after {mode} on the fresh buffers")
del fresh
torch.cuda.empty_cache()
measure("after freeing them")
