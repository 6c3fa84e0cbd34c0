#!/usr/bin/env python
"""Column-major corpus sequences on the device: GB/s (algorithmic bytes of the row-major
kernel; ATAX/BATAX need two passes over a transposed operand) + a launch-shape sweep of the
new rank-2 + row-dot pass."""
import ctypes, itertools, sys
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import _native, spec as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
lib = _native.load()
torch.cuda.set_device(0)
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
rnd = lambda *s: torch.rand(*s, dtype=torch.float64, device="cuda") * 2 - 1

def timed(fn, reps=7):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return sorted(ts)[len(ts) // 2]

SA, SB = rnd(n, n), torch.empty(n, n, dtype=torch.float64, device="cuda")
v = [rnd(n) for _ in range(7)]
x, w = torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")
def rank2():
    _native.check(lib.bto_rank2_rowdot_async(P(SA), P(v[0]), P(v[1]), P(v[2]), P(v[3]), P(v[4]), 0.3, P(v[5]),
                                             P(SB), P(x), n, n, st))
def colsum():
    _native.check(lib.bto_colsum_axpz_async(P(SB), P(x), 0.7, None, P(w), n, n, st))
print(f"n={n}")
for rows, minb, gps in itertools.product((8, 16), (1, 2), (1, 2, 4, 8)):
    try:
        _native.set_tuning(mv_rows=rows, mv_minb=minb, grid_per_sm=gps)
        t = timed(rank2)
        print(f"rank2_rowdot rows={rows:2d} minb={minb} grid/SM={gps}: {t*1e3:8.3f} ms {16.0*n*n/t/1e9:7.0f} GB/s", flush=True)
    except Exception as e:
        print("skip", rows, minb, gps, str(e)[:60])
_native.set_tuning(mv_rows=0, mv_minb=0, grid_per_sm=0)
t1, t2 = timed(rank2), timed(colsum)
print(f"defaults: rank2_rowdot {t1*1e3:.3f} ms ({16.0*n*n/t1/1e9:.0f} GB/s), colsum {t2*1e3:.3f} ms ({8.0*n*n/t2/1e9:.0f} GB/s); "
      f"GEMVER column-major {24.0*n*n/(t1+t2)/1e9:.0f} GB/s")
# whole sequences through the Python entry (device tensors, F-ordered)
for name in ("bicgk", "atax", "gesummv", "gemver"):
    g = S.infer_shapes(S.parse_kernel(S.CORPUS[name].replace("matrix(row)", "matrix(column)")))
    k = bto.gpu_kernel(g)
    ext = {"M": n, "N": n}
    inputs = {}
    for iname, decl in g.spec.inputs:
        if decl.kind == "scalar": inputs[iname] = 0.5
        elif decl.kind == "matrix": inputs[iname] = SA.t()
        else: inputs[iname] = v[0]
    t = timed(lambda: bto.run_kernel(bto.library_path(), k, g, inputs, ext), reps=5)
    print(f"{name:8s} column-major via run_kernel: {t*1e3:8.3f} ms  {_native.bytes_min(name, n, n)/t/1e9:7.0f} GB/s (row-major minimum bytes)")
