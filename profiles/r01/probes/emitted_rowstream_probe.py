#!/usr/bin/env python
"""Row-streaming (emitted) vs strip-tiled (hand-written) N-products at bench sizes."""
import json, sys, tempfile
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cost, cuemit
irs = json.loads((REPO / "tests/golden/organisms.json").read_text())
for name, n in (("gesummv", 24576), ("gesummv", 32768), ("dgemv", 32768), ("dgemv", 16384)):
    typed = bto.load_graph(name)
    ext = {"M": n, "N": n}
    fused = cost.measure_empirical(cost.GpuVariant(name), typed, ext, reps=7)
    best = None
    for tune in ({}, {"jam": 8, "unroll": 2}, {"jam": 4, "unroll": 4, "threads": 512, "minb": 1}, {"jam": 2, "unroll": 4}, {"jam": 8, "unroll": 4, "minb": 1}):
        k = cuemit.emit_cuda(irs[name][0], **tune)
        lib = cuemit.NvccToolchain().compile(k.source, tempfile.mkdtemp(), name="k")
        inputs = bto.gen_inputs(typed, ext, seed=7)
        dev = {a: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for a, v in inputs.items()}
        t = cuemit.time_emitted(lib, k, irs[name][0], dev, ext, reps=7)
        if best is None or t < best[0]: best = (t, tune)
        del dev
    nbytes = bto._native.bytes_min(name, n, n)
    print(f"{name} n={n}: hand-written {fused.total*1e3:.3f} ms ({nbytes/fused.total/1e9:.0f} GB/s)  emitted best {best[0]*1e3:.3f} ms ({nbytes/best[0]/1e9:.0f} GB/s) {best[1]}  [{irs[name][0]['organism']}]", flush=True)
