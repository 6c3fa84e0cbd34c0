#!/usr/bin/env python
"""Specs outside the hand-written set: fused emitted code (stored organisms of
tests/golden/noncorpus.json) against the statement-by-statement executor:  noncorpus_probe.py [n]"""
import json, sys, tempfile, time
from pathlib import Path
import numpy as np
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cuemit, spec as S
from paper_1205_1098_b200.generic import run_generic

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
stored = json.loads((REPO / "tests/golden/noncorpus.json").read_text())
tc = cuemit.NvccToolchain(cache_dir=tempfile.mkdtemp())
for key, entry in stored.items():
    typed = S.infer_shapes(S.parse_kernel(entry["spec"]))
    ext = {e: (n * n // 8 if len(typed.extent_names) == 1 else n) for e in typed.extent_names}
    inputs = bto.gen_inputs(typed, ext, seed=1)
    dev = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in inputs.items()}
    kernel = cuemit.emitted_kernel_for(typed, toolchain=tc, ir=entry["ir"])
    path, emitted, ir = cuemit.emitted_entry(kernel.source)
    t_emit = cuemit.time_emitted(path, emitted, ir, dev, ext, reps=5)
    run_generic(typed, dev, ext); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter(); run_generic(typed, dev, ext); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    a = bto.run_kernel(bto.library_path(), kernel, typed, dev, ext)
    b = run_generic(typed, dev, ext)
    err = bto.max_rel_error(a, {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in b.items()})
    print(f"{key:14s} {ext}  emitted {t_emit*1e3:9.3f} ms   generic {best*1e3:9.3f} ms   x{best/t_emit:6.2f}   "
          f"agree {err:.1e}   {ir['organism']}", flush=True)
