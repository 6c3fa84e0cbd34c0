#!/usr/bin/env python
"""Launch the matrix sequences at one mid size (for ncu launch lists):  mid_kernel.py 4096 3"""
import sys
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native  # noqa: E402
from paper_1205_1098_b200.sharded import GpuShardOps  # noqa: E402

n, reps = int(sys.argv[1]), int(sys.argv[2])
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    _native.set_tuning(**{k: int(v)})
torch.cuda.set_device(0)
ops = GpuShardOps()
A = torch.rand(n, n, dtype=torch.float64, device="cuda")
B = torch.rand(n, n, dtype=torch.float64, device="cuda")
v = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(8)]
o = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
torch.cuda.synchronize()
for _ in range(reps):
    ops.bicgk(A, v[0], v[1], o[0], o[1])
    ops.atax(A, v[0], o[0])
    ops.gesummv(0.5, 0.25, A, B, v[0], o[0])
    ops.gemver(A, v[0], v[1], v[2], v[3], 0.5, 0.25, v[4], v[5], B, o[0], o[1])
torch.cuda.synchronize()
print("ok")
