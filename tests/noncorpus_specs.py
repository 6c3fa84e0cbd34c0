"""Kernels outside the hand-written set: non-corpus specs and corpus kernels with mixed orientations."""

SPECS = {
    "vsub": "VSUB in: a : vector(column), b : vector(column) out: c : vector(column) { c = a - b }",
    "twomv": "TWOMV in: A : matrix(row), B : matrix(row), x : vector(column), y : vector(column) "
             "out: z : vector(column) { z = A' * x + B' * y }",
    "chain": "CHAIN in: alpha : scalar, beta : scalar, x : vector(column), y : vector(column) "
             "out: w : vector(column) { w = alpha * beta * x + y - beta * x }",
    "dotscale": "DOTSCALE in: x : vector(column), y : vector(column) out: z : vector(column), "
                "s : scalar { s = x' * y  z = s * x - y }",
    "rank1": "RANK1 in: A : matrix(row), u : vector(column), v : vector(column), "
             "x : vector(column) out: C : matrix(row), y : vector(column) "
             "{ C = A + u * v'  y = C * x }",
    "colmajor": "COLMAJOR in: A : matrix(column), x : vector(column), w : vector(column) "
                "out: y : vector(column), z : vector(column) { y = A * x  z = A' * w + x }",
    "mixed": "MIXED in: A : matrix(row), B : matrix(column), x : vector(column), gamma : scalar "
             "out: C : matrix(row), y : vector(column) { C = A - gamma * B  y = gamma * C * x }",
    "gram": "GRAM in: A : matrix(row), x : vector(column), lam : scalar out: y : vector(column) "
            "{ y = A' * (A * x) + lam * x }",
    # corpus kernels with MIXED orientations (the hand-written sequences cover all-row / all-column)
    "gemver_mixed": "GEMVER in: A : matrix(row), u1 : vector(column), v1 : vector(column), u2 : vector(column), v2 : vector(column), alpha : scalar, beta : scalar, y : vector(column), z : vector(column) out: B : matrix(column), x : vector(column), w : vector(column) { B = ((A + (u1 * v1')) + (u2 * v2'))  x = (((beta * B') * y) + z)  w = ((alpha * B) * x) }",
    "gesummv_mixed": "GESUMMV in: alpha : scalar, beta : scalar, A : matrix(row), B : matrix(column), x : vector(column) out: y : vector(column) { y = (((alpha * A) * x) + ((beta * B) * x)) }",
}

EXTENTS = [(1, 1), (7, 50), (300, 129), (513, 1026)]
