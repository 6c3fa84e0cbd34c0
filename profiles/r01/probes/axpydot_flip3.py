#!/usr/bin/env python
"""Is the 'fast state' tied to the last ALLOCATED or the last WRITTEN buffer?"""
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
bufs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(8)]
order = [int(x) for x in sys.argv[1].split(",")]
for i in order:
    bufs[i].uniform_(-1, 1)
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
print("fill order", order, " ".join(f"set{sys.argv[2][i]}={run([4 * int(sys.argv[2][i]) + k for k in range(4)]):.0f}" for i in range(len(sys.argv[2]))))
