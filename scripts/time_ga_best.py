#!/usr/bin/env python
"""Emit and time (on the GPU) the organisms stored by scripts/ga_on_gpu_model.py."""
import json, sys
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cuemit
data = json.loads((REPO / "profiles/r01/ga_best_irs.json").read_text())
for name, d in data.items():
    typed = bto.load_graph(name)
    entries = [("max_fuse", d["max_fuse"]), ("ga", d["ga"])] + [("alt", a) for a in d.get("alternatives", [])]
    for tag, e in entries:
        rep = cuemit.measure_empirical_ir(e["ir"], typed, d["extents"], reps=3)
        print(f"{name:8s} {tag:8s} model {e['model_ms']:8.3f} ms  measured "
              f"{rep.total*1e3 if not rep.failed else float('nan'):8.3f} ms  {e['organism'][:90]} {rep.diagnostic or ''}", flush=True)
