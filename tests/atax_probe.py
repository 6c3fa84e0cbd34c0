#!/usr/bin/env python
"""Fused ATAX: correctness across cluster sizes (against the oracle: test infrastructure, hence under tests/)
+ timing at the bench size (run on a B200)."""
from __future__ import annotations

import statistics
import sys
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))
import oracle_lib  # noqa: E402
import paper_1205_1098_b200 as bto  # noqa: E402
from paper_1205_1098_b200 import _native  # noqa: E402

g = bto.load_graph("atax")
k = bto.gpu_kernel(g)


def run(A, x):
    return bto.run_kernel(bto.library_path(), k, g, {"A": A, "x": x},
                          {"M": A.shape[0], "N": A.shape[1]})["y"]


def main():
    torch.cuda.set_device(0)
    bad = 0
    for (m, n) in [(2048, 1024), (8, 2), (1, 4096), (100, 514), (333, 8192), (64, 16390),
                   (1000, 4098), (37, 32768), (5000, 1026)]:
        inputs = bto.gen_inputs(g, {"M": m, "N": n}, seed=m + n)
        want = oracle_lib.oracle_run("atax", inputs, {"M": m, "N": n}, threads=8)["y"]
        A, x = torch.from_numpy(inputs["A"]).cuda(), torch.from_numpy(inputs["x"]).cuda()
        for C in (0, 1, 2, 4, 8, 16):
            for S, R, L in ((0, 0, 0), (2, 0, 0), (0, 1, 0), (4, 1, 0)):
                _native.set_tuning(atax_cluster=C, atax_stages=S, atax_rows=R, atax_fused=1)
                got = run(A, x).cpu().numpy()
                err = float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1.0)))
                flag = "" if err < 1e-11 else "  <-- BAD"
                bad += err >= 1e-11 or not np.isfinite(err)
                print(f"M={m:6d} N={n:6d} C={C:2d} S={S} R={R} L={L} err={err:.2e}{flag}", flush=True)
    print("correctness failures:", bad)
    n = 32768
    gen = torch.Generator(device="cuda").manual_seed(0)
    A = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    _native.set_tuning(atax_fused=0)
    ref = run(A, x)
    lib = _native.load()
    import ctypes
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _native.set_tuning(debug=1)
    cfgs = [(0, 0, 0, 0, 0)]
    for C in (4, 8, 16):
        for R in (0, 1):
            for S in (0, 2, 3):
                cfgs.append((1, C, S, R, 0))
    for fused, C, S, R, L in cfgs:
        _native.set_tuning(atax_fused=fused, atax_cluster=C, atax_stages=S, atax_rows=R)
        got = run(A, x)
        err = float(torch.max(torch.abs(got - ref) / torch.clamp(torch.abs(ref), min=1.0)))
        evs = []
        for _ in range(13):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _native.check(lib.bto_atax_async(A.data_ptr(), x.data_ptr(), y.data_ptr(), n, n, st))
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in evs[3:])
        print(f"bench fused={fused} C={C:2d} S={S} R={R} L={L}: {ms:.4f} ms  "
              f"{(8.0 * n * n + 16 * n) / ms / 1e6:7.1f} GB/s  err vs two-pass {err:.2e}", flush=True)


if __name__ == "__main__":
    main()
