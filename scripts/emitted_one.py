#!/usr/bin/env python
"""Run ONE emitted organism a few times (ncu target): emitted_one.py bicgk 0 8192 [jam=4 unroll=2 threads=256 blocks=592]"""
import json, sys, tempfile
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cuemit
name, idx, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
tune = {k: int(v) for k, v in (a.split("=") for a in sys.argv[4:])}
blocks = tune.pop("blocks", cuemit.DEFAULT_BLOCKS)
irs = json.loads((REPO / "tests/golden/organisms.json").read_text())
ir = irs[name][idx]
typed = bto.load_graph(name)
ext = {"M": n * n // 8} if typed.extent_names == ("M",) else {"M": n, "N": n}
kernel = cuemit.emit_cuda(ir, blocks=blocks, **tune)
tc = cuemit.NvccToolchain(template=cuemit.DEFAULT_TEMPLATE.replace("-O3", "-O3 -lineinfo"))
lib = tc.compile(kernel.source, Path(tempfile.mkdtemp()), name=name)
inputs = bto.gen_inputs(typed, ext, seed=1)
dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in inputs.items()}
t = cuemit.time_emitted(lib, kernel, ir, dev, ext, reps=3)
print(f"{name}[{idx}] n={n}: {t*1e3:.3f} ms")
