#!/usr/bin/env python
"""Fit cuemit.EmitModel's coefficients to measured organism timings (least squares on the
log error):  fit_emit_model.py [profiles/r01/organism_times.json]"""
import json, sys
from dataclasses import replace
from pathlib import Path
import numpy as np
from scipy.optimize import minimize
from scipy.stats import spearmanr
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1205_1098_b200 import cuemit
path = Path(sys.argv[1]) if len(sys.argv) > 1 else REPO / "profiles/r01/organism_times.json"
IRS = json.loads((REPO / "tests/golden/organisms.json").read_text())
rows = json.loads(path.read_text())
names = ["cta_gbs", "launch_us", "step_us", "free_step_us", "trip_us", "jam_trip_us", "rmw_trip_us",
         "stmt_us", "free_stmt_us", "alloc_us"]
base = cuemit.EmitModel()
meas = np.array([r["seconds"] for r in rows])

def predict(model):
    return np.array([cuemit.estimate_cost_ir(IRS[r["kernel"]][r["index"]], {"M": r["M"], "N": r["N"]}, model).total
                     for r in rows])

def loss(x):
    model = replace(base, **{n: float(np.exp(v)) for n, v in zip(names, x)})
    return float(np.mean(np.log(predict(model) / meas) ** 2))

x0 = np.log([max(getattr(base, n), 1e-3) for n in names])     # (zero coefficients: start small, not at -inf)
res = minimize(loss, x0, method="Nelder-Mead", options={"maxiter": 1500, "xatol": 1e-3, "fatol": 1e-5})
model = replace(base, **{n: float(np.exp(v)) for n, v in zip(names, res.x)})
pred = predict(model)
le = np.abs(np.log(pred / meas))
print({n: round(getattr(model, n), 4) for n in names})
print("spearman", round(spearmanr(pred, meas).correlation, 4), "median |log err|", round(float(np.median(le)), 3),
      "rms", round(float(np.sqrt(np.mean(le ** 2))), 3))
