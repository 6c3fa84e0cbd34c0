#!/usr/bin/env python
"""Does AXPYDOT's speed depend on WHICH 1 GiB buffers it streams (physical placement)?"""
import ctypes, random, sys
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native
lib = _native.load()
torch.cuda.set_device(0)
n = 1 << 27
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
bufs = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 24)]
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
    return ts[len(ts) // 2]
print("addresses (GiB):", [round(b.data_ptr() / 2**30, 3) for b in bufs])
order = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 3, 4, 5, 0]
for k in order:
    ix = [4 * k, 4 * k + 1, 4 * k + 2, 4 * k + 3]
    ms = run(ix)
    free, total = torch.cuda.mem_get_info()
    print(f"set {k} buffers {ix}: {ms:.4f} ms {32.0 * n / ms / 1e6:7.0f} GB/s", flush=True)
sys.exit(0)
# read-only and write-only rates per buffer (copy kernel via torch)
for i in (0, 5, 11, 17, 23):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.sum(bufs[i]); a.record(); s = torch.sum(bufs[i]); b.record(); b.synchronize()
    print(f"buffer {i}: torch.sum {8.0 * n / a.elapsed_time(b) / 1e6:7.0f} GB/s")
