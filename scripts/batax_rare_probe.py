#!/usr/bin/env python
"""Hunt for the non-finite BATAX result of the round-2 fuzz (633 x 8502, atax_per_sm=2, atax_cluster=9):
the same call many times with allocator churn in between; prints where the bad columns are and
where the operands live."""
import sys
from pathlib import Path
import numpy as np
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import _native

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
g = bto.load_graph("batax")
ext = {"M": 633, "N": 8502}
kernel = bto.gpu_kernel(g)
_native.set_tuning(atax_per_sm=2, atax_cluster=9, atax_fused=1)
inputs = bto.random_inputs(g, ext, seed=4321)
dev = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in inputs.items()}
ref = (dev["A"].t() @ (dev["A"] @ dev["x"])) * inputs["beta"]
print("A at", hex(dev["A"].data_ptr()), "x at", hex(dev["x"].data_ptr()))
bad = 0
shown = 0
for i in range(reps):
    if i % 7 == 0:
        junk = torch.rand(1 + (i * 7919) % 3000000, dtype=torch.float64, device="cuda")
        del junk
    y = bto.run_kernel(bto.library_path(), kernel, g, dev, ext)["y"]
    err = ((y - ref).abs() / ref.abs().clamp(min=1.0))
    wrong = ~(err < 1e-10)
    if bool(wrong.any()):
        bad += 1
        if shown < 6:
            shown += 1
            idx = torch.nonzero(wrong).flatten()
            runs = []
            lo = prev = int(idx[0])
            for v in idx[1:].tolist():
                if v != prev + 1:
                    runs.append((lo, prev)); lo = v
                prev = v
            runs.append((lo, prev))
            print(f"call {i}: y at {hex(y.data_ptr())}: {idx.numel()} wrong columns, runs {runs[:8]}, "
                  f"values {y[idx[:3]].tolist()}", flush=True)
print(f"{_native.launch_plan()}: {reps} repeats, {bad} wrong")
_native.set_tuning(atax_per_sm=1, atax_cluster=0)
