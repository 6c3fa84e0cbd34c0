"""numpy evaluation of a kernel spec AS WRITTEN -- TEST INFRASTRUCTURE.

Restates the semantics of the reference's interpreter (interp.py:20-129: tagged
scalar/col/row/mat values, np.dot / @ / np.outer, statement by statement) over
this repository's AST, for kernels outside the corpus, where the C oracle has no
function.  Pinned by tests/test_generic.py against the golden O1 outputs of the
reference for every corpus kernel.
"""
from __future__ import annotations

import numpy as np


def evaluate(spec, inputs: dict, dtype=np.float64) -> dict:
    """`dtype=np.longdouble` gives an extended-precision evaluation: the yardstick for reductions
    over 10^5..10^6 terms, where the C oracle's one-after-the-other sums carry more rounding
    error than the tolerance allows either side."""
    env = {}
    for name, decl in spec.inputs:
        v = inputs[name]
        if decl.kind == "scalar":
            env[name] = ("scalar", dtype(v))
        elif decl.kind == "vector":
            env[name] = ("col" if decl.orientation == "column" else "row", np.asarray(v, dtype=dtype))
        else:
            env[name] = ("mat", np.asarray(v, dtype=dtype))

    def ev(e):
        if e[0] == "var":
            return env[e[1]]
        if e[0] == "t":
            k, d = ev(e[1])
            return {"col": "row", "row": "col", "mat": "mat"}[k], (d.T if k == "mat" else d)
        (lk, ld), (rk, rd) = ev(e[1]), ev(e[2])
        if e[0] in "+-":
            assert lk == rk
            return lk, (ld + rd if e[0] == "+" else ld - rd)
        if lk == "scalar" or rk == "scalar":
            return (rk if lk == "scalar" else lk), ld * rd
        if lk == "row" and rk == "col":
            return "scalar", dtype(np.dot(ld, rd))
        if lk == "col" and rk == "row":
            return "mat", np.outer(ld, rd)
        if lk == "mat" and rk == "col":
            return "col", ld @ rd
        raise ValueError(f"cannot multiply {lk} by {rk}")

    for target, expr in spec.statements:
        env[target] = ev(expr)
    return {n: (float(env[n][1]) if d.kind == "scalar" else np.array(env[n][1], dtype=np.float64))
            for n, d in spec.outputs}
