#!/usr/bin/env python
"""Host-side cost of one library call (wall clock, no sync inside the loop)."""
import ctypes, sys, time
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native
from paper_1205_1098_b200.sharded import GpuShardOps
torch.cuda.set_device(0)
lib = _native.load(); ops = GpuShardOps()
n = 4096
x = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(4)]
A = torch.rand(256, 512, dtype=torch.float64, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: ctypes.c_void_p(t.data_ptr())
B_ = torch.empty_like(A); xo = torch.empty(512, dtype=torch.float64, device="cuda"); wo = torch.empty(256, dtype=torch.float64, device="cuda")
def bench(label, fn, reps=3000):
    for _ in range(50): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{label:34s} issue {1e6*(t1-t0)/reps:6.2f} us/call   incl. drain {1e6*(t2-t0)/reps:6.2f} us/call")
bench("ctypes bto_abi_version", lambda: lib.bto_abi_version())
bench("ctypes bto_get_tuning", lambda: lib.bto_get_tuning(b"mv_rows"))
bench("torch add (1 kernel)", lambda: torch.add(x[0], x[1], out=x[2]))
bench("raw bto_vadd_async", lambda: lib.bto_vadd_async(P(x[0]), P(x[1]), P(x[2]), P(x[3]), n, st))
a, b, c, d = P(x[0]), P(x[1]), P(x[2]), P(x[3])
bench("raw bto_vadd_async (args cached)", lambda: lib.bto_vadd_async(a, b, c, d, n, st))
bench("ops.bicgk 256x512 (2 kernels)", lambda: ops.bicgk(A, x[0][:512], x[1][:256], x[2][:256], x[3][:512]))
bench("ops.atax 256x512 (2 kernels)", lambda: ops.atax(A, x[0][:512], x[3][:512]))
f = ops.bind("bicgk", A, x[0][:512], x[1][:256], x[2][:256], x[3][:512])
bench("ops.bind('bicgk') 256x512 (2 kernels)", f)
g = ops.bind("gemver", A, x[1][:256], x[0][:512], x[1][:256], x[0][:512], 0.5, 0.25, x[2][:256], x[3][:512],
             torch.empty_like(A), torch.empty(512, dtype=torch.float64, device="cuda"), torch.empty(256, dtype=torch.float64, device="cuda"))
bench("ops.bind('gemver') 256x512", g)
bench("ops.gemver 256x512", lambda: ops.gemver(A, x[1][:256], x[0][:512], x[1][:256], x[0][:512], 0.5, 0.25, x[2][:256], x[3][:512], B_, xo, wo))
