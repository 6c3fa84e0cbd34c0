#!/usr/bin/env python
"""Emitted ATAX (two strided loops per row batch): L2 footprint (CTAs x jam x row) against barrier rate."""
import itertools, json, sys, tempfile
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cuemit
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ir = json.loads((REPO / "tests/golden/organisms.json").read_text())["atax"][0]
typed = bto.load_graph("atax")
ext = {"M": n, "N": n}
inputs = bto.gen_inputs(typed, ext, seed=1)
dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in inputs.items()}
grid = [dict(jam=j, unroll=u, threads=t, blocks=b, minb=m, bypass_l1=bp)
        for (j, t, b, m), u, bp in itertools.product(
            [(2, 256, 592, 2), (4, 256, 592, 2), (4, 512, 296, 1), (8, 512, 296, 1), (8, 1024, 148, 1),
             (16, 1024, 148, 1), (4, 1024, 148, 1), (2, 512, 296, 2), (8, 256, 296, 2), (4, 256, 296, 2)],
            (2, 4), (0, 1))]
work = Path(tempfile.mkdtemp()); tc = cuemit.NvccToolchain()
def build(i):
    cfg = dict(grid[i]); blocks = cfg.pop("blocks")
    k = cuemit.emit_cuda(ir, blocks=blocks, **cfg)
    return i, k, tc.compile(k.source, work, name=f"atax_{i}")
with ThreadPoolExecutor(max_workers=12) as pool:
    built = list(pool.map(build, range(len(grid))))
rows = []
for i, k, lib in built:
    try:
        t = cuemit.time_emitted(lib, k, ir, dev, ext, reps=5)
    except Exception as e:
        print("fail", grid[i], e); continue
    rows.append((t, grid[i]))
for t, cfg in sorted(rows, key=lambda r: r[0])[:12]:
    print(f"{t*1e3:.3f} ms  {8.0*n*n/t/1e9:6.0f} GB/s  {cfg}", flush=True)
