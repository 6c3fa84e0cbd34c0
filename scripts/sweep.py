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


PIECES = ("gemver_pass1", "gemver_pass2", "tonly", "dgemv")
PIECE_BYTES = {"gemver_pass1": 16.0, "gemver_pass2": 8.0, "tonly": 8.0, "dgemv": 8.0}


def launch_piece(suite, name):
    """Single passes of the matrix engine on the suite's buffers (n = 32768)."""
    import ctypes
    lib, n = _native.load(), suite.n
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if name == "gemver_pass1":
        rc = lib.bto_gemver_pass1_async(P(suite.A), P(suite.vecM[1]), P(suite.vecN[1]),
                                        P(suite.vecM[2]), P(suite.vecN[2]), P(suite.vecM[0]),
                                        P(suite.Bm), P(suite.colsum), n, n, st)
    elif name == "tonly":
        rc = lib.bto_gemver_pass1_async(P(suite.A), None, None, None, None, P(suite.vecM[0]),
                                        None, P(suite.colsum), n, n, st)
    elif name == "gemver_pass2":
        rc = lib.bto_gemver_pass2_async(P(suite.Bm), P(suite.vecN[0]), 0.5, P(suite.w), n, n, st)
    else:
        rc = lib.bto_dgemv_async(0.5, P(suite.A), P(suite.vecN[0]), 0.25, P(suite.vecM[0]),
                                 P(suite.w), n, n, st)
    _native.check(rc)


THRASH = None      # a launch closure run (untimed) before every timed rep
SUSTAIN = 0.0      # seconds of back-to-back launches before timing (power-capped state)


def time_kernel(suite, name, reps):
    if name in PIECES:
        orig = suite.launch
        launch = lambda _n: launch_piece(suite, name)
    else:
        launch = suite.launch
    if SUSTAIN > 0:
        import time
        t_end = time.perf_counter() + SUSTAIN       # reach the power-capped steady state
        while time.perf_counter() < t_end:
            for _ in range(20):
                launch(name)
            torch.cuda.synchronize()
    for _ in range(3):
        launch(name)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    for a, b in evs:
        if THRASH is not None:
            THRASH()
        a.record()
        launch(name)
        b.record()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    return statistics.median(ms), min(ms)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernels", default=",".join(SUITE))
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--sustain", type=float, default=0.0,
                    help="seconds of back-to-back launches before timing each config")
    ap.add_argument("--thrash", action="store_true",
                    help="run GEMVER (16 GiB of other traffic) before every timed rep, as in the suite")
    ap.add_argument("--out", default=str(REPO / "gpurun_out" / "sweep.json"))
    args = ap.parse_args()
    kernels = tuple(args.kernels.split(","))
    torch.cuda.set_device(0)
    _native.load()
    global THRASH, SUSTAIN
    SUSTAIN = args.sustain
    suite = Suite(torch, 0, 1, tuple(set(k for k in kernels if k not in PIECES) | {"gemver"}))
    if args.thrash:
        THRASH = lambda: suite.launch("gemver")
    peak, _ = measured_peak()
    rows = []
    mv_cfgs = [(8, 1), (16, 1), (32, 1), (8, 2)]
    grids = [0, 2, 4, 8, 16] if not args.quick else [0, 4]
    minbs = [1, 2, 3, 4, 6] if not args.quick else [1, 3]
    for name in kernels:
        if name == "axpydot":
            cfgs = [dict(vec_unroll=u, vec_grid_per_sm=g)
                    for u, g in itertools.product([1, 2, 4], [0, 2, 4, 8, 16])]
        else:
            cfgs = [dict(mv_rows=r, mv_vec=v, grid_per_sm=g, mv_minb=b)
                    for (r, v), g, b in itertools.product(mv_cfgs, grids, minbs)]
            if name == "atax":
                cfgs = [dict(atax_cluster=c, atax_rows=r, atax_stages=st)
                        for c, r, st in itertools.product([4, 8, 16], [0, 1], [0, 2, 3])]
        for cfg in cfgs:
            _native.set_tuning(**cfg)
            try:
                med, best = time_kernel(suite, name, args.reps)
            except Exception as exc:
                print(name, cfg, "FAILED", exc)
                continue
            nbytes = PIECE_BYTES[name] * 32768.0 ** 2 if name in PIECES else bytes_min(name, *BENCH[name])
            gbs = nbytes / (med * 1e-3) / 1e9
            rows.append({"kernel": name, **cfg, "ms_median": med, "ms_min": best,
                         "gbs": gbs, "frac": gbs / peak})
            print(f"{name:8s} {cfg} median {med:8.4f} ms  min {best:8.4f} ms  "
                  f"{gbs:7.1f} GB/s  {100 * gbs / peak:5.1f}%", flush=True)
        _native.set_tuning(mv_rows=0, mv_vec=0, grid_per_sm=0, mv_minb=0, vec_unroll=2, vec_grid_per_sm=0,
                           atax_cluster=0, atax_rows=0, atax_stages=0)
    Path(args.out).parent.mkdir(exist_ok=True)
    Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
