#!/usr/bin/env python
"""Run the emitted CUDA of selected organisms a few times (target for ncu launch lists):
   emitted_kernels.py 8192 [plain]"""
import json, sys, tempfile
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cuemit
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
optimize = "plain" not in sys.argv[2:]
irs = json.loads((REPO / "tests/golden/organisms.json").read_text())
best = json.loads((REPO / "profiles/r01/ga_best_irs.json").read_text())
todo = [("axpydot", irs["axpydot"][0]), ("bicgk", irs["bicgk"][0]), ("atax", irs["atax"][0]),
        ("gesummv", irs["gesummv"][0]), ("gemver", best["gemver"]["alternatives"][1]["ir"])]
work = Path(tempfile.mkdtemp())
for name, ir in todo:
    typed = bto.load_graph(name)
    ext = {"M": n * n // 8} if typed.extent_names == ("M",) else {"M": n, "N": n}
    kernel = cuemit.emit_cuda(ir, optimize=optimize)
    lib = cuemit.NvccToolchain().compile(kernel.source, work, name=name)
    inputs = bto.gen_inputs(typed, ext, seed=1)
    dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in inputs.items()}
    for _ in range(3):
        cuemit.run_emitted(lib, kernel, ir, dev, ext)
    torch.cuda.synchronize()
    print("ran", name, ir["organism"], flush=True)
