#!/usr/bin/env python
"""Measure every fixture organism's emitted CUDA (tests/golden/organisms.json) on the GPU.
Output: gpurun_out/organism_times.json  [{kernel, index, organism, M, N, seconds}]"""
import json, sys, tempfile
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cuemit
irs = json.loads((REPO / "tests/golden/organisms.json").read_text())
sizes = [int(a) for a in sys.argv[1:]] or [2048]
wd = Path(tempfile.mkdtemp())
tc = cuemit.NvccToolchain()
jobs = [(name, i, ir) for name, lst in irs.items() for i, ir in enumerate(lst)]
def build(job):
    name, i, ir = job
    k = cuemit.emit_cuda(ir)
    return job, k, tc.compile(k.source, wd, name=f"{name}_{i}")
with ThreadPoolExecutor(max_workers=16) as pool:
    built = list(pool.map(build, jobs))
rows = []
for n in sizes:
    for (name, i, ir), kernel, path in built:
        typed = bto.load_graph(name)
        ext = {"M": n * n} if typed.extent_names == ("M",) else {"M": n, "N": n}
        inputs = bto.gen_inputs(typed, ext, seed=1)
        dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in inputs.items()}
        best = cuemit.time_emitted(path, kernel, ir, dev, ext, reps=3)
        rows.append({"kernel": name, "index": i, "organism": ir["organism"], "M": ext["M"],
                     "N": ext.get("N", 1), "seconds": best})
        print(f"n={n} {name:8s} #{i:2d} {best*1e3:9.3f} ms  {ir['organism'][:70]}", flush=True)
(REPO / "gpurun_out").mkdir(exist_ok=True)
(REPO / "gpurun_out" / "organism_times.json").write_text(json.dumps(rows, indent=1))
