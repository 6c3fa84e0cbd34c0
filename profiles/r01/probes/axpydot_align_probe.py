#!/usr/bin/env python
"""Does the relative placement of AXPYDOT's four 1 GiB streams matter (DRAM channel / bank phase)?"""
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
pool = torch.empty(5 * n + (1 << 24), dtype=torch.float64, device="cuda")
pool.uniform_(-1, 1)
beta = torch.empty(1, dtype=torch.float64, device="cuda")
def run(delta_elems):
    offs = [k * (n + delta_elems) for k in range(4)]
    w, v, u, z = (pool[o:o + n] for o in offs)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    fn = lambda: _native.check(lib.bto_axpydot_async(P(w), P(v), P(u), 0.37, P(z), P(beta), n, st))
    for _ in range(3): fn()
    ts = []
    for _ in range(9):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]
print("base address % 2MiB:", pool.data_ptr() % (1 << 21))
for d in (0, 2, 32, 64, 128, 256, 512, 1024, 4096, 1 << 14, 1 << 16, 1 << 17, 1 << 18, 1 << 20, (1 << 18) + 512, 3 << 16):
    ms = run(d)
    print(f"stream spacing 1 GiB + {d * 8:9d} B: {ms:7.4f} ms  {32.0 * n / ms / 1e6:7.0f} GB/s", flush=True)
