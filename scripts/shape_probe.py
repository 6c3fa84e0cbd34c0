#!/usr/bin/env python
"""GB/s of the matrix sequences on extreme aspect ratios (tall-skinny, short-wide), ~2 GiB each."""
import sys
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native
from paper_1205_1098_b200.sharded import GpuShardOps
torch.cuda.set_device(0)
ops = GpuShardOps()
shapes = [(1 << 22, 32), (1 << 22, 64), (1 << 21, 100), (1 << 20, 256), (1 << 19, 500), (1 << 18, 1000),
          (16384, 16384), (1000, 1 << 18), (64, 1 << 22), (8, 1 << 24), (3, 1 << 26)]
args = [a for a in sys.argv[1:] if "=" not in a]
for kv in (a for a in sys.argv[1:] if "=" in a):           # tuning keys, e.g. grid_per_sm=8
    k, v = kv.split("=")
    _native.set_tuning(**{k: int(v)})
if args:
    shapes = [tuple(int(x) for x in a.split("x")) for a in args]
def timed(fn, reps=5):
    for _ in range(2): fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b) * 1e-3)
    return sorted(ts)[len(ts) // 2]
for m, n in shapes:
    A = torch.rand(m, n, dtype=torch.float64, device="cuda")
    B = torch.empty(m, n, dtype=torch.float64, device="cuda")
    vn = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(4)]
    vm = [torch.rand(m, dtype=torch.float64, device="cuda") for _ in range(4)]
    on, om = torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(m, dtype=torch.float64, device="cuda")
    res = {}
    # GB/s of the algorithmic minimum (vectors included: at M = 8 they are a fifth of it)
    bm = lambda k: _native.bytes_min(k, m, n)
    res["bicgk"] = bm("bicgk") / timed(lambda: ops.bicgk(A, vn[0], vm[0], om, on))
    res["atax"] = bm("atax") / timed(lambda: ops.atax(A, vn[0], on))
    B.copy_(A)
    res["gesummv"] = bm("gesummv") / timed(lambda: ops.gesummv(0.5, 0.25, A, B, vn[0], om))
    res["gemver"] = bm("gemver") / timed(lambda: ops.gemver(A, vm[0], vn[0], vm[1], vn[1], 0.5, 0.25, vm[2], vn[2], B, on, om))
    print(f"{m:9d} x {n:9d}: " + "  ".join(f"{k} {v/1e9:6.0f}" for k, v in res.items()) + "  GB/s", flush=True)
    del A, B
