#!/usr/bin/env python
"""8 x 1 GiB buffers; AXPYDOT on buffers 0-3 is slow until <action>; which actions flip it?"""
import ctypes, sys
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native
lib = _native.load()
torch.cuda.set_device(0)
n = 1 << 27
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
action = sys.argv[1]
if action == "ws_first":                       # library workspace allocated BEFORE the big buffers
    t = torch.rand(4096, dtype=torch.float64, device="cuda"); o = torch.empty(4096, dtype=torch.float64, device="cuda")
    b0 = torch.empty(1, dtype=torch.float64, device="cuda")
    _native.check(lib.bto_axpydot_async(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(t.data_ptr()), 0.5,
                                        ctypes.c_void_p(o.data_ptr()), ctypes.c_void_p(b0.data_ptr()), 4096, st))
    torch.cuda.synchronize()
bufs = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(8)]
beta = torch.empty(1, dtype=torch.float64, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
def run(ix, reps=8):
    w, v, u, z = (bufs[i] for i in ix)
    fn = lambda: _native.check(lib.bto_axpydot_async(P(w), P(v), P(u), 0.37, P(z), P(beta), n, st))
    for _ in range(3): fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return 32.0 * n / ts[len(ts) // 2] / 1e6
before = run([0, 1, 2, 3])
if action == "sum7": torch.sum(bufs[7])
elif action == "sum4": torch.sum(bufs[4])
elif action == "sum7tail": torch.sum(bufs[7][-(1 << 24):])       # last 128 MiB written
elif action == "sum7head": torch.sum(bufs[7][: 1 << 24])
elif action == "write_scratch": s = torch.zeros(1 << 26, dtype=torch.float64, device="cuda"); torch.sum(s)
elif action == "read567": [torch.sum(bufs[i]) for i in (5, 6, 7)]
elif action == "axpy4567": run([4, 5, 6, 7])
elif action == "axpy_w7": run([7, 1, 2, 3])
elif action == "axpy_z7": run([0, 1, 2, 7])
elif action == "vadd4567":
    _native.check(lib.bto_vadd_async(P(bufs[4]), P(bufs[5]), P(bufs[6]), P(bufs[7]), n, st))
elif action == "axpy7small":
    m = 1 << 20
    _native.check(lib.bto_axpydot_async(P(bufs[7]), P(bufs[7][m:]), P(bufs[7][2 * m:]), 0.37, P(bufs[7][3 * m:]), P(beta), m, st))
elif action == "axpy7tail":
    m = 1 << 20
    _native.check(lib.bto_axpydot_async(P(bufs[7][-4 * m:]), P(bufs[7][-3 * m:]), P(bufs[7][-2 * m:]), 0.37, P(bufs[7][-m:]), P(beta), m, st))
elif action == "axpy4only":
    run([4, 1, 2, 3])
elif action == "sleep":
    import time; torch.cuda.synchronize(); time.sleep(1.0)
torch.cuda.synchronize()
after = run([0, 1, 2, 3])
print(f"{action:14s} before {before:6.0f}  after {after:6.0f} GB/s", flush=True)
