#!/usr/bin/env python
"""Mid-size (launch-bound) behaviour: per-call time issued eagerly back to back and replayed
from a CUDA graph of 20 calls (no host cost), against the HBM-ideal time."""
import json
import sys
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import _native  # noqa: E402
from paper_1205_1098_b200.sharded import GpuShardOps  # noqa: E402

torch.cuda.set_device(0)
lib = _native.load()
ops = GpuShardOps()
PEAK = 6551.0
sizes = [int(a) for a in sys.argv[1:] if a.isdigit()] or [1024, 2048, 3072, 4096, 6144, 8192]
# variants: name:key=value,key=value ... (bto_set_tuning keys), e.g.
#   split:join_fused=0 fused:join_fused=2 rows:join_fused=2,rowstream=2,rowstream_min_n=1024
VARIANTS = [a for a in sys.argv[1:] if ":" in a] or ["default:"]
DEFAULTS = {}
rows = []
for variant in VARIANTS:
  vname, _, kvs = variant.partition(":")
  tune = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in kvs.split(",") if kv}
  for k in tune:
      DEFAULTS.setdefault(k, _native.get_tuning(k))
  _native.set_tuning(**DEFAULTS)
  _native.set_tuning(**tune)
  for n in sizes:
      A = torch.rand(n, n, dtype=torch.float64, device="cuda")
      B = torch.rand(n, n, dtype=torch.float64, device="cuda")
      v = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(8)]
      o = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
      big = torch.rand(4, n * n // 8, dtype=torch.float64, device="cuda")
      beta = torch.empty(1, dtype=torch.float64, device="cuda")
      calls = {
          "axpydot": (lambda: ops.axpydot(big[0], big[1], big[2], 0.3, big[3], beta), 32.0 * (n * n // 8)),
          "bicgk": (lambda: ops.bicgk(A, v[0], v[1], o[0], o[1]), 8.0 * n * n),
          "atax": (lambda: ops.atax(A, v[0], o[0]), 8.0 * n * n),
          "gesummv": (lambda: ops.gesummv(0.5, 0.25, A, B, v[0], o[0]), 16.0 * n * n),
          "gemver": (lambda: ops.gemver(A, v[0], v[1], v[2], v[3], 0.5, 0.25, v[4], v[5], B, o[0], o[1]),
                     24.0 * n * n),
      }
      for name, (fn, nbytes) in calls.items():
          for _ in range(5):
              fn()
          torch.cuda.synchronize()
          l0 = _native.kernel_launches(); fn(); launches = _native.kernel_launches() - l0
          a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
          a.record()
          for _ in range(100):
              fn()
          b.record()
          torch.cuda.synchronize()
          us_eager = a.elapsed_time(b) * 1e3 / 100
          side = torch.cuda.Stream()
          g = torch.cuda.CUDAGraph()
          with torch.cuda.stream(side):
              fn()
              side.synchronize()
              with torch.cuda.graph(g, stream=side):
                  for _ in range(20):
                      fn()
          g.replay(); torch.cuda.synchronize()
          a.record()
          for _ in range(5):
              g.replay()
          b.record()
          torch.cuda.synchronize()
          us_graph = a.elapsed_time(b) * 1e3 / 100
          ideal = nbytes / PEAK / 1e3
          rows.append({"variant": vname, "kernel": name, "n": n, "launches": launches, "us_eager": us_eager, "us_graph": us_graph,
                       "us_ideal": ideal})
          print(f"{vname:8s} n={n:5d} {name:8s} launches={launches} eager {us_eager:7.1f} us  graph {us_graph:7.1f} us  "
                f"ideal {ideal:6.1f} us  graph/ideal {us_graph / ideal:5.2f}", flush=True)
(REPO / "gpurun_out").mkdir(exist_ok=True)
(REPO / "gpurun_out" / "midsize_probe.json").write_text(json.dumps(rows, indent=1))
