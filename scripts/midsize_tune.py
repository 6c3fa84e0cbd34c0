#!/usr/bin/env python
"""Which launch variant is fastest at mid sizes?  Every variant of cost.variant_space, timed as a
CUDA graph of 20 calls (no host cost), n = 1024 .. 8192:  midsize_tune.py [kernel ...] [n ...]"""
import json
import sys
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native, cost  # noqa: E402
from paper_1205_1098_b200.sharded import GpuShardOps  # noqa: E402

torch.cuda.set_device(0)
_native.load()
ops = GpuShardOps()
kernels = [a for a in sys.argv[1:] if not a.isdigit()] or ["bicgk", "gemver", "gesummv", "atax"]
sizes = [int(a) for a in sys.argv[1:] if a.isdigit()] or [1024, 2048, 4096, 8192]
EXTRA = {"bicgk": [(("mv_rows", r), ("mv_vec", v), ("mv_minb", mb), ("grid_per_sm", g))
                   for r, v in ((8, 1), (8, 2), (16, 1)) for mb in (2, 4) for g in (1, 2, 4)]}


def graph_us(fn):
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        fn()
        side.synchronize()
        with torch.cuda.graph(g, stream=side):
            for _ in range(20):
                fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / 20)
    return best


rows = []
for n in sizes:
    A = torch.rand(n, n, dtype=torch.float64, device="cuda")
    B = torch.rand(n, n, dtype=torch.float64, device="cuda")
    v = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(8)]
    o = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
    calls = {
        "bicgk": lambda: ops.bicgk(A, v[0], v[1], o[0], o[1]),
        "atax": lambda: ops.atax(A, v[0], o[0]),
        "gesummv": lambda: ops.gesummv(0.5, 0.25, A, B, v[0], o[0]),
        "gemver": lambda: ops.gemver(A, v[0], v[1], v[2], v[3], 0.5, 0.25, v[4], v[5], B, o[0], o[1]),
    }
    for name in kernels:
        space = [cost.GpuVariant(name)] + cost.variant_space(name) + \
            [cost.GpuVariant(name, t) for t in EXTRA.get(name, [])]
        seen, results = set(), []
        for var in space:
            if var.key() in seen:
                continue
            seen.add(var.key())
            saved = {k: _native.get_tuning(k) for k, _ in var.tuning}
            try:
                _native.set_tuning(**dict(var.tuning))
                us = graph_us(calls[name])
            except _native.BtoError:
                continue
            finally:
                _native.set_tuning(**saved)
            results.append((us, var.key()))
        results.sort()
        default = next(us for us, k in results if k == cost.GpuVariant(name).key())
        print(f"n={n} {name}: default {default:.1f} us; best " +
              "; ".join(f"{us:.1f} {k}" for us, k in results[:4]), flush=True)
        rows.append({"n": n, "kernel": name, "default_us": default, "ranked": results[:10]})
(REPO / "gpurun_out").mkdir(exist_ok=True)
(REPO / "gpurun_out" / "midsize_tune.json").write_text(json.dumps(rows, indent=1))
