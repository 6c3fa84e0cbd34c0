#!/usr/bin/env python
"""Randomised differential test: every corpus kernel, random extents (biased to strip / tile
edges), random launch tunables, device and host operands, against the CPU oracle.
   fuzz_parity.py [seconds] [seed]"""
import math, random, sys, time
from pathlib import Path
import numpy as np
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO)); sys.path.insert(0, str(REPO / "tests"))   # test infrastructure: may use the oracle
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import _native
import oracle_lib
import np_interp
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
ONLY = sys.argv[3].split(",") if len(sys.argv) > 3 else None       # e.g. atax,batax: hunt in one family
oracle = oracle_lib.load_oracle() if hasattr(oracle_lib, "load_oracle") else oracle_lib
ELEMENTWISE = {"axpydot": ("z",), "vadd": ("x",), "waxpby": ("w",), "gemver": ("B",)}
def extent():
    r = rng.random()
    if r < 0.25: return rng.choice([1, 2, 3, 7, 8, 9, 15, 16, 17, 31, 32, 33, 63, 64, 65])
    if r < 0.5: return max(1, rng.choice([256, 512, 1024, 1536, 2048]) + rng.randint(-3, 3))
    if r < 0.85: return rng.randint(1, 3000)
    if r < 0.95: return rng.randint(3000, 20000)
    return rng.choice([303106, 606210, 700000, 1200002])      # thousands of strips: the column-direct path
t_end = time.time() + budget
cases = fails = 0
while time.time() < t_end:
    name = rng.choice(sorted(ONLY or bto.CORPUS))
    g = bto.load_graph(name)
    m, n = extent(), extent()
    if name in ("atax", "batax") and rng.random() < 0.5:
        # rows long enough for every cluster size of the single-pass kernel (slices of 5..8 iterations)
        m, n = rng.randint(1, 700), 2 * rng.randint(3000, 22000) + rng.choice([0, 0, 0, 1])
    if m * n > 3e7:
        if n > 300000: m = max(1, int(3e7 // n))             # keep the very wide shapes wide
        else: n = max(1, int(3e7 // m))
    ext = {"M": m * n} if g.extent_names == ("M",) else {"M": m, "N": n}
    tune = dict(mv_rows=rng.choice([0, 0, 8, 16, 32]), mv_vec=rng.choice([0, 0, 1, 2]),
                grid_per_sm=rng.choice([0, 0, 1, 2, 4, 8]), mv_minb=rng.choice([0, 0, 1, 2, 4]),
                skinny=rng.choice([1, 1, 0]), vec_unroll=rng.choice([1, 2, 4]), atax_fused=rng.choice([1, 1, 0]),
                direct_cols=rng.choice([1, 1, 0]), midsize=rng.choice([1, 1, 0]), atax_per_sm=rng.choice([1, 1, 2]),
                atax_cluster=rng.choice([0, 0, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 16]), rowstream=rng.choice([1, 1, 0, 2]))
    _native.set_tuning(**tune)
    if rng.random() < 0.5:
        _native.poison_shared_memory()      # NaN patterns in every SM's shared memory before the call
        _native.poison_workspace()          # ... and in the partial-sum workspace
    inputs = bto.random_inputs(g, ext, seed=cases)
    want = oracle.oracle_run(name, inputs, ext, threads=rng.choice([1, 4, 8]))
    host = rng.random() < 0.3
    from paper_1205_1098_b200.colmajor import COLMAJOR_SEQUENCES
    colmajor = name in COLMAJOR_SEQUENCES and rng.random() < 0.25
    if colmajor:        # same logical kernel on F-ordered operands: fused, roles swapped (colmajor.py)
        from paper_1205_1098_b200 import spec as bspec
        g = bspec.infer_shapes(bspec.parse_kernel(bspec.CORPUS[name].replace("matrix(row)", "matrix(column)")))
    if host:
        got = bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, inputs, ext)
    else:
        dev = {k: (torch.from_numpy(np.ascontiguousarray(v)).cuda() if isinstance(v, np.ndarray) else v) for k, v in inputs.items()}
        for k, t in list(dev.items()):          # some vectors at an odd 8-byte offset
            if hasattr(t, "dim") and t.dim() == 1 and rng.random() < 0.2:
                shifted = torch.empty(t.numel() + 1, dtype=torch.float64, device="cuda")[1:]
                shifted.copy_(t)
                dev[k] = shifted
        got = bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, dev, ext)
        got = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in got.items()}
    if max(ext.values()) >= 8192:
        # sums of 3*10^4..10^6 cancelling terms: the oracle adds them one after the other (like the
        # reference's C) and is itself 1.5-2e-11 off at N = 40000 for ATAX's two chained reductions
        # (numpy's pairwise sums: 1.3e-12), more beyond; judge the GPU against an extended-precision
        # evaluation, and the oracle too (loosely: it must still be the same function).  Vector
        # kernels too: a one-thread oracle adds AXPYDOT's 4.4 M products one after the other, ~4e-11
        # absolute, which the metric |g - e| / max(|e|, 1) shows whenever the dot happens to be small.
        exact = np_interp.evaluate(bto.load_graph(name).spec, inputs, dtype=np.longdouble)
        assert bto.max_rel_error(want, exact) < 1e-9, (name, ext)
        reductions = {k: v for k, v in exact.items() if k not in ELEMENTWISE.get(name, ())}
        want = dict(want, **reductions)
    err = bto.max_rel_error(got, want)
    tol = 1e-12 * max(1.0, math.log2(max(ext.values())))
    bad = not (err <= tol) or any(np.any(np.isnan(np.asarray(got[o]))) for o in want)
    for o in ELEMENTWISE.get(name, ()):
        bad = bad or not np.array_equal(np.asarray(got[o]), np.asarray(want[o]))
    cases += 1
    if bad:
        fails += 1
        # what kind of failure: NaNs (where, how many, on which side), and does it repeat?
        for o in want:
            a, b = np.asarray(got[o], dtype=np.float64).ravel(), np.asarray(want[o], dtype=np.float64).ravel()
            na, nb = np.flatnonzero(~np.isfinite(a)), np.flatnonzero(~np.isfinite(b))
            d = np.abs(a - b) / np.maximum(np.abs(b), 1.0)
            print(f"   {o}: non-finite in result {na.size} (first {na[:4].tolist()}), in oracle {nb.size}; "
                  f"worst element {int(np.nanargmax(d)) if d.size else -1} of {a.size}", flush=True)
        if not host:
            again = 0
            for _ in range(10):
                rep = bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, dev, ext)
                rep = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in rep.items()}
                again += int(not (bto.max_rel_error(rep, want) <= tol))
            print(f"   the same call repeated 10 times: {again} mismatches", flush=True)
        print("MISMATCH", f"case {cases - 1}", name, ext, tune, "host" if host else "device", "colmajor" if colmajor else "",
              f"err={err:.3e}", flush=True)
_native.set_tuning(mv_rows=0, mv_vec=0, grid_per_sm=0, mv_minb=0, skinny=1, vec_unroll=2, atax_fused=1,
                   direct_cols=1, midsize=1, atax_per_sm=1, atax_cluster=0, rowstream=1)
print(f"{cases} cases, {fails} mismatches")
sys.exit(1 if fails else 0)
