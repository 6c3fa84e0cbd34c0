#!/usr/bin/env python
"""Emitted ATAX / BATAX / BiCGK (row read twice) in cluster mode against the plain mapping and the
hand-written sequence:  emit_cluster_sweep.py [n=32768]"""
import json, sys, tempfile
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cost, cuemit

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
irs = json.loads((REPO / "tests/golden/organisms.json").read_text())
work = Path(tempfile.mkdtemp()); tc = cuemit.NvccToolchain()
for name in ("atax", "batax"):
    ir = next(i for i in irs[name] if "{_i{_j 1}{_j 2}}" in i["organism"] and i["organism"].startswith("{_{p(i)}"))
    typed = bto.load_graph(name)
    ext = {"M": n, "N": n}
    inputs = bto.gen_inputs(typed, ext, seed=7)
    dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in inputs.items()}
    nbytes = bto._native.bytes_min("atax", n, n)
    hand = cost.measure_empirical(cost.GpuVariant(name), typed, ext, reps=5)
    print(f"{name} n={n}: hand-written {hand.total*1e3:.3f} ms {nbytes/hand.total/1e9:.0f} GB/s", flush=True)
    cfgs = [dict(cluster=0), dict(cluster=8, cluster_min_bytes=0), dict(cluster=4, cluster_min_bytes=0),
            dict(cluster=8, cluster_min_bytes=0, cluster_jam=2, cluster_minb=4),
            dict(cluster=4, cluster_min_bytes=0, cluster_jam=2, cluster_minb=2, cluster_threads=512)]
    if "--full" in sys.argv:
        for C in (8, 4):
            for jam in (2, 4, 8):
                for minb, threads in ((2, 256), (3, 256), (4, 256), (1, 512), (2, 512)):
                    cfgs.append(dict(cluster=C, cluster_min_bytes=0, cluster_jam=jam, cluster_minb=minb,
                                     cluster_threads=threads))
    for tag, cfg in enumerate(cfgs):
        try:
            k = cuemit.emit_cuda(ir, **cfg)
            lib = tc.compile(k.source, work, name=f"{name}_{tag}")
            t = cuemit.time_emitted(lib, k, ir, dev, ext, reps=5)
            print(f"  {cfg}: {t*1e3:8.3f} ms {nbytes/t/1e9:7.0f} GB/s  ({hand.total/t:.2f} of hand-written)", flush=True)
        except Exception as exc:
            print(f"  {cfg}: FAILED {str(exc)[:200]}", flush=True)
