#!/usr/bin/env python
"""Per-call wall time of the host-pointer (pinned) calls of the suite against the PCIe floor."""
import ctypes, sys, time
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native
lib = _native.load()
torch.cuda.set_device(0)
n, g, a = 32768, 24576, 1 << 27
pin = lambda c: torch.empty(c, dtype=torch.float64, pin_memory=True)
big_in, big_out = pin(n * n), pin(n * n)
big_in.uniform_(-1, 1)
vec = [pin(n).uniform_(-1, 1) for _ in range(8)]
outv = [pin(n) for _ in range(3)]
scalar = pin(1)
P = lambda t: ctypes.c_void_p(t.data_ptr())
calls = {
 "axpydot": (lambda: lib.axpydot(P(big_in[:a]), P(big_in[a:2*a]), P(big_in[2*a:3*a]), 0.37, P(big_out[:a]), P(scalar), a), 24.0*a, 8.0*a),
 "bicgk": (lambda: lib.bicgk(P(big_in), P(vec[0]), P(vec[1]), P(outv[0]), P(outv[1]), n, n), 8.0*n*n, 0),
 "atax": (lambda: lib.atax(P(big_in), P(vec[0]), P(outv[0]), n, n), 8.0*n*n, 0),
 "gesummv": (lambda: lib.gesummv(0.61, -0.27, P(big_in[:g*g]), P(big_in[g*g:2*g*g] if 2*g*g <= n*n else big_in[:g*g]), P(vec[0]), P(outv[0]), g, g), 16.0*g*g, 0),
 "gemver": (lambda: lib.gemver(P(big_in), P(vec[1]), P(vec[2]), P(vec[3]), P(vec[4]), 0.83, -0.41, P(vec[5]), P(vec[6]), P(big_out), P(outv[1]), P(outv[2]), n, n), 8.0*n*n, 8.0*n*n),
}
# raw PCIe rate for reference
dev = torch.empty(n * n // 4, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); dev.copy_(big_in[: n * n // 4], non_blocking=True); torch.cuda.synchronize()
    rate = 8.0 * dev.numel() / (time.perf_counter() - t0) / 1e9
print(f"raw pinned H2D: {rate:.1f} GB/s")
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    _native.set_tuning(**{k: int(v)})
for name, (fn, h2d, d2h) in calls.items():
    if sys.argv[1:] and name not in ("axpydot", "gemver"):
        continue
    fn(); _native.check()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); fn(); _native.check(); ts.append(time.perf_counter() - t0)
    t = sorted(ts)[1]
    floor = max(h2d, d2h) / (rate * 1e9)
    print(f"{name:8s} {t*1e3:7.1f} ms   floor {floor*1e3:7.1f} ms   ratio {t/floor:5.3f}   H2D {h2d/t/1e9:5.1f} GB/s", flush=True)
