#!/usr/bin/env python
"""Generate tests/golden/noncorpus.json from the REFERENCE (build container only).

For kernels OUTSIDE the hand-written set -- non-corpus specs and corpus kernels with MIXED matrix
orientations -- record what `cuemit.emitted_kernel_for` derives where the reference is importable:
the loop IR of the organism the reference's MFGA finds best under the GPU cost model, plus O1
outputs of the reference's interpreter (interp.py:100) on the reference's random inputs for a few
extents, so that the GPU box (no reference there) can emit, compile, run and check the fused code.

Run:  python tests/golden/make_noncorpus.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))

import matfuse  # noqa: E402
from matfuse import reference_evaluate  # noqa: E402
from matfuse.graph import build_dataflow, infer_types  # noqa: E402
from matfuse.runtime import random_inputs  # noqa: E402

from paper_1205_1098_b200 import cuemit  # noqa: E402
from paper_1205_1098_b200 import spec as S  # noqa: E402
from noncorpus_specs import SPECS, EXTENTS  # noqa: E402

out = {}
for key, text in SPECS.items():
    ours = S.parse_kernel(text)
    g = infer_types(build_dataflow(matfuse.parse_kernel(S.format_kernel(ours))))
    assert S.parse_kernel(S.format_kernel(ours)) == ours, key
    ir = cuemit.ir_for_spec(g)
    cases = []
    for (m, n) in EXTENTS:
        ext = {e: (m if e == "M" else n) for e in g.extent_names}
        inputs = random_inputs(g, ext, seed=m + n)
        want = reference_evaluate(g.spec, inputs)
        # the generator must be the one the tests re-run (same draws, same order)
        mine = __import__("paper_1205_1098_b200").random_inputs(S.infer_shapes(ours), ext, seed=m + n)
        for k, v in inputs.items():
            assert np.array_equal(np.asarray(v), np.asarray(mine[k])), (key, k)
        cases.append({"ext": ext, "seed": m + n,
                      "out": {k: (float(v) if np.ndim(v) == 0 else np.asarray(v).ravel()[:64].tolist())
                              for k, v in want.items()},
                      "sum": {k: float(np.sum(np.asarray(v, dtype=np.float64))) for k, v in want.items()}})
    out[key] = {"spec": text, "ir": ir, "cases": cases}
    print(f"{key:12s} {ir['organism']}")
(HERE / "noncorpus.json").write_text(json.dumps(out, separators=(",", ":")))
