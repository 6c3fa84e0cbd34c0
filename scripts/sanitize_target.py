#!/usr/bin/env python
"""Small end-to-end run of every sequence and path, sized for compute-sanitizer."""
import sys
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto  # noqa: E402
from paper_1205_1098_b200 import _native  # noqa: E402

torch.cuda.set_device(0)
_native.load()
shapes = [(37, 29), (300, 1026), (129, 515), (64, 4100)]
for name in bto.CORPUS:
    g = bto.load_graph(name)
    k = bto.gpu_kernel(g)
    for (m, n) in shapes:
        ext = {"M": m * n} if g.extent_names == ("M",) else {"M": m, "N": n}
        inp = bto.gen_inputs(g, ext, seed=1)
        bto.run_kernel(bto.library_path(), k, g, inp, ext)                       # host pointers
        dev = {a: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for a, v in inp.items()}
        bto.run_kernel(bto.library_path(), k, g, dev, ext)                       # device pointers
for c in (1, 2, 4, 8, 9, 16):
    _native.set_tuning(atax_cluster=c)
    g = bto.load_graph("atax")
    inp = bto.gen_inputs(g, {"M": 50, "N": 2050}, seed=2)
    dev = {a: torch.from_numpy(v).cuda() for a, v in inp.items()}
    bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, dev, {"M": 50, "N": 2050})
_native.set_tuning(atax_cluster=0, host_panel_mib=1)
g = bto.load_graph("gemver")
inp = bto.gen_inputs(g, {"M": 2100, "N": 2050}, seed=3)
bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, inp, {"M": 2100, "N": 2050})   # host pipeline
torch.cuda.synchronize()
print("sanitize target ok")
