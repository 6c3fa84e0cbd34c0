#!/usr/bin/env python
"""From the fast state: which neighbouring kernel slows AXPYDOT down?"""
import ctypes, sys
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native
from paper_1205_1098_b200.sharded import GpuShardOps
lib = _native.load()
torch.cuda.set_device(0)
n = 1 << 27
m = 32768
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ops = GpuShardOps()
A = torch.empty(m, m, dtype=torch.float64, device="cuda")
B = torch.empty(m, m, dtype=torch.float64, device="cuda")
vv = [torch.empty(m, dtype=torch.float64, device="cuda") for _ in range(10)]
bufs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(4)]
for t in [A] + vv + bufs[::-1]:            # last written: bufs[0], which AXPYDOT sweeps
    t.uniform_(-1, 1)
beta = torch.empty(1, dtype=torch.float64, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
axpy = lambda: _native.check(lib.bto_axpydot_async(P(bufs[0]), P(bufs[1]), P(bufs[2]), 0.37, P(bufs[3]), P(beta), n, st))
others = {
    "bicgk": lambda: ops.bicgk(A, vv[0], vv[1], vv[2], vv[3]),
    "atax": lambda: ops.atax(A, vv[0], vv[3]),
    "gesummv": lambda: ops.gesummv(0.5, 0.25, A[:24576 * 24576 // m], A[:24576 * 24576 // m], vv[0], vv[2][:24576 * 24576 // m]),
    "gemver": lambda: ops.gemver(A, vv[0], vv[1], vv[2], vv[3], 0.5, 0.25, vv[4], vv[5], B, vv[6], vv[7]),
    "torch_fill_B": lambda: B.fill_(1.0),
    "torch_copy_A_to_B": lambda: B.copy_(A),
}
def batch(seq, reps=12):
    for _ in range(2):
        for f in seq: f()
    evs = []
    for _ in range(reps):
        for f in seq:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record()
            if f is axpy: evs.append((a, b))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return 32.0 * n / ts[len(ts) // 2] / 1e6
print(f"axpydot alone: {batch([axpy]):.0f} GB/s", flush=True)
for name, fn in others.items():
    print(f"[{name}, axpydot] alternating: {batch([fn, axpy]):.0f} GB/s;  axpydot alone afterwards: {batch([axpy]):.0f}", flush=True)
print(f"[bicgk, atax, gesummv, gemver, axpydot]: {batch([others['bicgk'], others['atax'], others['gesummv'], others['gemver'], axpy]):.0f}")
