#!/usr/bin/env python
"""Run the REFERENCE's MFGA (build container only) with the organism-level GPU cost model
as its fitness; snapshot the winners' loop IR so a GPU box can emit and time them."""
import json, sys
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
from matfuse import SearchConfig, cached, contract_arrays, lower, max_fuse, run_strategy
from matfuse.corpus import load_graph
from matfuse.fuse import canonical_key
from paper_1205_1098_b200 import cuemit

n = 4096
out = {}
for name in ("axpydot", "bicgk", "atax", "gesummv", "gemver"):
    g = load_graph(name)
    ext = {"M": n * n} if g.extent_names == ("M",) else {"M": n, "N": n}
    fitness = cached(cuemit.AnalyticOrganismCost(g, ext))
    res = run_strategy("mfga", g, SearchConfig(core_count=8, generations=20, seed=0), fitness)
    seed_org = max_fuse(g, 8)
    out[name] = {
        "extents": ext,
        "ga": {"organism": canonical_key(res.best), "model_ms": res.best_fitness * 1e3,
               "ir": cuemit.ir_from_matfuse(contract_arrays(lower(res.best, g)))},
        "max_fuse": {"organism": canonical_key(seed_org), "model_ms": fitness(seed_org).total * 1e3,
                     "ir": cuemit.ir_from_matfuse(contract_arrays(lower(seed_org, g)))},
        "evaluations": res.evaluations,
    }
    print(f"{name:8s} evals {res.evaluations:4d}  GA best {res.best_fitness*1e3:8.3f} ms {canonical_key(res.best)}")
    print(f"{'':8s}            max-fuse {out[name]['max_fuse']['model_ms']:8.3f} ms {canonical_key(seed_org)}")
# hand-picked alternatives recorded earlier (GEMVER's row-partitioned organisms) stay, re-priced
path = REPO / "profiles" / "r01" / "ga_best_irs.json"
if path.exists():
    for name, entry in json.loads(path.read_text()).items():
        for alt in entry.get("alternatives", []):
            alt["model_ms"] = cuemit.estimate_cost_ir(alt["ir"], out[name]["extents"]).total * 1e3
            out[name].setdefault("alternatives", []).append(alt)
path.write_text(json.dumps(out, separators=(",", ":")))
