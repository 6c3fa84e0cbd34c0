"""Corpus sequences on column-major operands, still fused.

A `matrix(column)` operand (lang.py:17-31; the reference hands the C function an
F-ordered buffer, runtime.py:92-95, and indexes it `i + j*M`, cemit.py:64-65) is,
as a buffer, the row-major TRANSPOSE `S` of the logical matrix.  With `A = S'`
every product swaps its kind -- `A x = S' x` is a weighted column sum of `S`,
`A' r = S r` a row dot -- so each corpus sequence maps onto the row-major fused
passes of the library with the operands' roles exchanged, and every matrix
element still crosses HBM the minimum number of times:

    BiCGK    q = A p, s = A' r         -> bicgk(S; p := r, r := p) with q, s exchanged    (1 pass)
    ATAX     y = A'(A x) = S (S' x)    -> dgemvt(S): t = S' x, then y = S t              (2 passes: the
    BATAX    y = beta A'(A x)             first product needs every row of S before the second starts)
    GESUMMV  y = alpha A x + beta B x  -> two column-sum passes, the second adding the first (1 pass each)
    DGEMV    z = alpha A x + beta y    -> t = y*beta, then z = (S' x)*alpha + t            (1 pass)
    DGEMVT   x = beta A' y + z,        -> dgemv(S) for x (row dots), column sums for w     (2 passes)
             w = alpha A x
    GEMVER   B = A + u1 v1' + u2 v2'   -> rank2_rowdot(S_A; v1,u1,v2,u2; y) writes S_B and x,
             x = beta B' y + z            then w = (S_B' x)*alpha                          (A 1x, B 1x + 1x)
             w = alpha B x

Each statement keeps the reference's rounding (one rounded operation per
statement, cemit.py:112-136), so `B`, and `x`/`w`/`y`/`z` given the same sums,
come out as the reference's would; sums differ by reduction order only.
Operands are torch CUDA tensors or numpy arrays of the LOGICAL shape; a tensor
that already is F-ordered (`S.t()`) is used in place.
"""
from __future__ import annotations

import ctypes

from . import _native

__all__ = ["COLMAJOR_SEQUENCES", "column_major_variant", "run_colmajor"]

#: corpus kernels with matrix operands (the vector-only ones have no storage order)
COLMAJOR_SEQUENCES = ("bicgk", "atax", "batax", "gesummv", "dgemv", "dgemvt", "gemver")


def column_major_variant(spec):
    """Name of the corpus kernel `spec` equals once every matrix is read as
    `matrix(row)` -- provided ALL its matrices are `matrix(column)`; else None."""
    from .spec import Decl, KernelSpec, UnsupportedKernelError, match_corpus
    mats = [d for _, d in tuple(spec.inputs) + tuple(spec.outputs) if d.kind == "matrix"]
    if not mats or any(d.orientation != "column" for d in mats):
        return None
    as_row = KernelSpec(
        spec.name,
        tuple((n, Decl(d.kind, "row") if d.kind == "matrix" else d) for n, d in spec.inputs),
        tuple((n, Decl(d.kind, "row") if d.kind == "matrix" else d) for n, d in spec.outputs),
        spec.statements)
    try:
        name = match_corpus(as_row)
    except UnsupportedKernelError:
        return None
    return name if name in COLMAJOR_SEQUENCES else None


def run_colmajor(name: str, graph, inputs: dict, extents: dict, stream=None) -> dict:
    """Run corpus kernel `name` whose matrices are all column-major.  `graph` is the
    TypedSpec of the caller's spec (its own identifier names, the corpus's argument order)."""
    import numpy as np
    import torch

    lib = _native.load()
    stream = stream or torch.cuda.current_stream()
    st = ctypes.c_void_p(stream.cuda_stream)
    spec = graph.spec
    on_gpu = any(hasattr(inputs.get(n), "is_cuda") and inputs[n].is_cuda for n, _ in spec.inputs)

    def P(t):
        return ctypes.c_void_p(t.data_ptr()) if t is not None else None

    def new(*shape):
        return torch.empty(*shape, dtype=torch.float64, device="cuda")

    vals = []
    for iname, decl in spec.inputs:
        if iname not in inputs:
            raise ValueError(f"missing input {iname!r}")
        v = inputs[iname]
        if decl.kind == "scalar":
            vals.append(float(v))
            continue
        want = tuple(int(extents[d]) for d in graph.dims[iname])
        if tuple(np.shape(v)) != want:
            raise ValueError(f"{iname}: expected shape {want}, got {tuple(np.shape(v))}")
        if hasattr(v, "is_cuda"):
            t = v.to("cuda", torch.float64)
        elif decl.kind == "matrix":
            # F-ordered host array = row-major transpose: copy that buffer, view it back
            t = _native.to_device(np.asarray(v, dtype=np.float64).T).t()
        else:
            t = _native.to_device(v)
        # the buffer the reference would pass: F-ordered logical matrix = row-major transpose
        vals.append(t.t().contiguous() if decl.kind == "matrix" else t.contiguous())
    M, N = int(extents[graph.extent_names[0]]), int(extents[graph.extent_names[1]])
    ck = _native.check
    outs = {}
    onames = [n for n, _ in spec.outputs]

    if name == "bicgk":
        S, p, r = vals
        q, s = new(M), new(N)
        ck(lib.bto_bicgk_async(P(S), P(r), P(p), P(s), P(q), N, M, st))        # S is N x M
        outs = {onames[0]: q, onames[1]: s}
    elif name in ("atax", "batax"):
        if name == "atax":
            S, x = vals
            beta = 1.0
        else:
            x, beta, S = vals
        t, y, zero = new(M), new(N), torch.zeros(M, dtype=torch.float64, device="cuda")
        # t = (S' x)*1 + 0 ; y = (S t)*beta   (BATAX: y = t1*beta, the reference's last statement)
        ck(lib.bto_dgemvt_async(beta, 1.0, P(S), P(x), P(zero), P(t), P(y), N, M, st))
        outs = {onames[0]: y}
    elif name == "gesummv":
        alpha, beta, SA, SB, x = vals
        t1, y = new(M), new(M)
        ck(lib.bto_colsum_axpz_async(P(SA), P(x), alpha, None, P(t1), N, M, st))   # t1 = t0*alpha
        ck(lib.bto_colsum_axpz_async(P(SB), P(x), beta, P(t1), P(y), N, M, st))    # y = t2*beta + t1
        # the reference adds t1 + t3 with t1 first; IEEE addition commutes, the bits are the same
        outs = {onames[0]: y}
    elif name == "dgemv":
        alpha, S, x, beta, yv = vals
        t2, z = new(M), new(M)
        ck(lib.bto_prim_axpby_async(beta, P(yv), 0.0, None, P(t2), M, 0, st))      # t2 = y*beta
        ck(lib.bto_colsum_axpz_async(P(S), P(x), alpha, P(t2), P(z), N, M, st))    # z = t0*alpha + t2
        outs = {onames[0]: z}
    elif name == "dgemvt":
        alpha, beta, S, yv, zv = vals
        x, w = new(N), new(M)
        ck(lib.bto_dgemv_async(beta, P(S), P(yv), 1.0, P(zv), P(x), N, M, st))     # x = (S y)*beta + z*1
        ck(lib.bto_colsum_axpz_async(P(S), P(x), alpha, None, P(w), N, M, st))     # w = (S' x)*alpha
        outs = {onames[0]: x, onames[1]: w}
    elif name == "gemver":
        SA, u1, v1, u2, v2, alpha, beta, yv, zv = vals
        SB, x, w = new(N, M), new(N), new(M)
        ck(lib.bto_rank2_rowdot_async(P(SA), P(v1), P(u1), P(v2), P(u2), P(yv), beta, P(zv),
                                      P(SB), P(x), N, M, st))
        ck(lib.bto_colsum_axpz_async(P(SB), P(x), alpha, None, P(w), N, M, st))
        outs = {onames[0]: SB.t(), onames[1]: x, onames[2]: w}                   # B: logical M x N, F-ordered
    else:
        raise ValueError(f"no column-major sequence for {name!r}")
    stream.synchronize()
    if on_gpu:
        return outs
    host = {}
    for k, v in outs.items():
        # a column-major matrix comes back F-ordered, like the reference's reshape(order="F")
        host[k] = _native.to_host(v.t()).T if (v.dim() == 2 and not v.is_contiguous()) else _native.to_host(v)
    return host
