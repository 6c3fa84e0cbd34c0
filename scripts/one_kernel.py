#!/usr/bin/env python
"""Launch one suite kernel a few times (for ncu captures):  one_kernel.py atax 6"""
import sys
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from bench import Suite  # noqa: E402
from paper_1205_1098_b200 import _native  # noqa: E402

name, reps = sys.argv[1], int(sys.argv[2])
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    _native.set_tuning(**{k: int(v)})
torch.cuda.set_device(0)
suite = Suite(torch, 0, 1, (name,))
for _ in range(reps):
    suite.launch(name)
torch.cuda.synchronize()
print("ok")
