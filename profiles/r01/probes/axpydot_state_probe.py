#!/usr/bin/env python
"""AXPYDOT runs at 6.3 or 7.0 TB/s depending on a device state: which? (time, clocks, neighbours)"""
import ctypes, sys, time
from pathlib import Path
import torch, pynvml
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native
from paper_1205_1098_b200.sharded import GpuShardOps
lib = _native.load()
torch.cuda.set_device(0)
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
def clocks():
    return (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
            pynvml.nvmlDeviceGetPowerUsage(h) // 1000)
n = 1 << 27
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
bufs = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(8)]
A = torch.rand(16384, 16384, dtype=torch.float64, device="cuda")
vv = [torch.rand(16384, dtype=torch.float64, device="cuda") for _ in range(4)]
beta = torch.empty(1, dtype=torch.float64, device="cuda")
ops = GpuShardOps()
P = lambda t: ctypes.c_void_p(t.data_ptr())
def axpy(k=0):
    _native.check(lib.bto_axpydot_async(P(bufs[k]), P(bufs[k + 1]), P(bufs[k + 2]), 0.37, P(bufs[k + 3]), P(beta), n, st))
def bicg():
    ops.bicgk(A, vv[0], vv[1], vv[2], vv[3])
def batch(label, seq, reps):
    evs = []
    for _ in range(reps):
        for name, fn in seq:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); evs.append((name, a, b))
    torch.cuda.synchronize()
    ax = [a.elapsed_time(b) for nme, a, b in evs if nme == "axpy"]
    print(f"{label:34s} first {ax[0]:.3f} last {ax[-1]:.3f} min {min(ax):.3f} max {max(ax):.3f} ms  clocks(sm,mem,W)={clocks()}", flush=True)
    return ax
torch.cuda.synchronize(); time.sleep(0.5)
print("idle clocks", clocks())
ax = batch("200 x axpy from idle", [("axpy", axpy)], 200)
print("   per-launch ms:", " ".join(f"{t:.3f}" for t in ax[:120:4]))
batch("50 x axpy again", [("axpy", axpy)], 50)
batch("50 x (bicgk, axpy)", [("bicg", bicg), ("axpy", axpy)], 50)
batch("50 x axpy after that", [("axpy", axpy)], 50)
batch("50 x axpy other buffers", [("axpy", lambda: axpy(4))], 50)
batch("25 x (axpy bufs0, axpy bufs4)", [("axpy", axpy), ("axpy", lambda: axpy(4))], 25)
time.sleep(1.0)
batch("50 x axpy after 1 s idle", [("axpy", axpy)], 50)
