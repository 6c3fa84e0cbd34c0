#!/usr/bin/env python
"""Time the emitted CUDA of the max-fuse organisms next to the hand-written sequences."""
import json, sys, tempfile
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cost, cuemit
irs = json.loads((REPO / "tests/golden/organisms.json").read_text())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
for name in bto.HOT_PATH:
    typed = bto.load_graph(name)
    ext = {"M": n * n} if typed.extent_names == ("M",) else {"M": n, "N": n}
    fused = cost.measure_empirical(cost.GpuVariant(name), typed, ext, reps=5)
    emitted = cuemit.measure_empirical_ir(irs[name][0], typed, ext, reps=3)
    plain = cuemit.measure_empirical_ir(irs[name][0], typed, ext, reps=3, optimize=False)
    import tempfile
    k2 = cuemit.emit_cuda(irs[name][0], bypass_l1=0)
    lib2 = cuemit.NvccToolchain().compile(k2.source, tempfile.mkdtemp(), name="nobypass")
    inputs = bto.gen_inputs(typed, ext, seed=7)
    dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in inputs.items()}
    t2 = cuemit.time_emitted(lib2, k2, irs[name][0], dev, ext, reps=3)
    print(f"{name:8s} emitted with L1-allocating loads: {t2*1e3:8.3f} ms", flush=True)
    unf = cuemit.measure_empirical_ir(irs[name][1], typed, ext, reps=1)
    nbytes = bto._native.bytes_min(name, ext["M"], ext.get("N", 1))
    print(f"{name:8s} n={n}: hand-written {fused.total*1e3:8.3f} ms ({nbytes/fused.total/1e9:6.0f} GB/s)   "
          f"emitted max-fuse {emitted.total*1e3:8.3f} ms ({nbytes/emitted.total/1e9:6.0f} GB/s)   "
          f"plain mapping {plain.total*1e3:8.3f} ms   "
          f"emitted unfused {unf.total*1e3:9.3f} ms  {emitted.diagnostic or ''} {unf.diagnostic or ''}", flush=True)

# GEMVER: the CPU max-fuse organism partitions columns; the row-partitioned ones the GA finds on
# the GPU model (profiles/r01/ga_best_irs.json) are the fair comparison
best = json.loads((REPO / "profiles/r01/ga_best_irs.json").read_text())
typed = bto.load_graph("gemver")
ext = {"M": n, "N": n}
nbytes = bto._native.bytes_min("gemver", n, n)
for entry in best["gemver"]["alternatives"]:
    ir = entry["ir"]
    e = cuemit.measure_empirical_ir(ir, typed, ext, reps=3)
    p = cuemit.measure_empirical_ir(ir, typed, ext, reps=3, optimize=False)
    print(f"gemver {ir['organism']}: emitted {e.total*1e3:8.3f} ms ({nbytes/e.total/1e9:6.0f} GB/s)  "
          f"plain {p.total*1e3:8.3f} ms {e.diagnostic or ''}", flush=True)
