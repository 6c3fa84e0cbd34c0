#!/usr/bin/env python
"""Sweep the emitter's tunables (jam, unroll, threads, blocks) on selected organisms:
   emit_sweep.py 8192"""
import itertools, json, sys, tempfile
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cuemit
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
irs = json.loads((REPO / "tests/golden/organisms.json").read_text())
best = json.loads((REPO / "profiles/r01/ga_best_irs.json").read_text())
todo = [("bicgk", irs["bicgk"][0]), ("atax", irs["atax"][0]), ("gesummv", irs["gesummv"][0]),
        ("gemver", best["gemver"]["alternatives"][1]["ir"])]
grid = [dict(jam=j, unroll=u, threads=256, blocks=b, minb=m) for j, u, m, b in
        itertools.product((2, 4, 8), (1, 2, 4), (2, 3, 4), (592, 1184))]
work = Path(tempfile.mkdtemp())
tc = cuemit.NvccToolchain()
rows = []
for name, ir in todo:
    typed = bto.load_graph(name)
    ext = {"M": n, "N": n}
    inputs = bto.gen_inputs(typed, ext, seed=1)
    dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in inputs.items()}
    nbytes = bto._native.bytes_min(name, n, n)
    def build(i):
        cfg = dict(grid[i]); blocks = cfg.pop("blocks")
        k = cuemit.emit_cuda(ir, blocks=blocks, **cfg)
        return i, k, tc.compile(k.source, work, name=f"{name}_{i}")
    with ThreadPoolExecutor(max_workers=12) as pool:
        built = list(pool.map(build, range(len(grid))))
    for i, k, lib in built:
        t = cuemit.time_emitted(lib, k, ir, dev, ext, reps=5)
        rows.append(dict(kernel=name, **grid[i], ms=t * 1e3, gbs=nbytes / t / 1e9))
    mine = sorted((r for r in rows if r["kernel"] == name), key=lambda r: r["ms"])
    for r in mine[:6] + mine[-2:]:
        print(r, flush=True)
(REPO / "gpurun_out").mkdir(exist_ok=True)
(REPO / "gpurun_out" / f"emit_sweep_{n}.json").write_text(json.dumps(rows, indent=1))
