#!/usr/bin/env python
"""Time every hot-path sequence at BASELINE bench sizes across launch tunables.

Run on a B200 (through gpurun); writes gpurun_out/sweep.json and prints a table.
    python scripts/sweep.py [--kernels bicgk,atax] [--reps 10] [--quick]
"""
from __future__ import annotations

import argparse
import itertools
import json
import statistics
import sys
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from bench import BENCH, SUITE, Suite, bytes_min, measured_peak  # noqa: E402
from paper_1205_1098_b200 import _native  # noqa: E402


def time_kernel(suite, name, reps):
    for _ in range(3):
        suite.launch(name)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    for a, b in evs:
        a.record()
        suite.launch(name)
        b.record()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    return statistics.median(ms), min(ms)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernels", default=",".join(SUITE))
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=str(REPO / "gpurun_out" / "sweep.json"))
    args = ap.parse_args()
    kernels = tuple(args.kernels.split(","))
    torch.cuda.set_device(0)
    _native.load()
    suite = Suite(torch, 0, 1, kernels)
    peak, _ = measured_peak()
    rows = []
    mv_cfgs = [(8, 1), (16, 1), (8, 2)]
    grids = [0, 1, 2, 3, 4, 6, 8] if not args.quick else [0, 2, 4]
    for name in kernels:
        if name == "axpydot":
            cfgs = [dict(vec_unroll=u, vec_grid_per_sm=g)
                    for u, g in itertools.product([1, 2, 4], [0, 2, 4, 8, 16])]
        else:
            cfgs = [dict(mv_rows=r, mv_vec=v, grid_per_sm=g)
                    for (r, v), g in itertools.product(mv_cfgs, grids)]
        for cfg in cfgs:
            _native.set_tuning(**cfg)
            try:
                med, best = time_kernel(suite, name, args.reps)
            except Exception as exc:
                print(name, cfg, "FAILED", exc)
                continue
            gbs = bytes_min(name, *BENCH[name]) / (med * 1e-3) / 1e9
            rows.append({"kernel": name, **cfg, "ms_median": med, "ms_min": best,
                         "gbs": gbs, "frac": gbs / peak})
            print(f"{name:8s} {cfg} median {med:8.4f} ms  min {best:8.4f} ms  "
                  f"{gbs:7.1f} GB/s  {100 * gbs / peak:5.1f}%", flush=True)
        _native.set_tuning(mv_rows=8, mv_vec=2, grid_per_sm=0, vec_unroll=4, vec_grid_per_sm=0)
    Path(args.out).parent.mkdir(exist_ok=True)
    Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
