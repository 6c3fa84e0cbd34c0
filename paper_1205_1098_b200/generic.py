"""Generic (unfused) executor: any valid kernel spec on the device.

The hand-written fused sequences cover the reference's corpus.  A spec outside
it is evaluated statement by statement with the unfused primitives of
`include/bto_b200.h` section 3c -- temporaries live in HBM, exactly what the
reference's unfused organism (`fuse.initial_forest`) does on the CPU -- so the
drop-in accepts the whole kernel language (`lang.py:17-31`), including
`matrix(column)` operands, not only the ten corpus kernels.

Evaluation order follows the reference's canonicalisation (graph.py:285-315):
scalar coefficients are carried past product chains and applied once, to the
vector result, so `beta * B' * y` never materialises a scaled matrix; sums scale
their operands and add with separately rounded operations (cemit.py:112-136).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _native
from .spec import KernelSpecError, TypedSpec

__all__ = ["run_generic", "GenericValue"]


@dataclass
class GenericValue:
    """A value on the device: `coef * data`, with `data` a contiguous fp64 CUDA
    tensor.  For a matrix `trans` says that `data` holds the TRANSPOSE of the
    logical matrix in row-major order (how a column-major operand is stored)."""
    kind: str                  # "scalar" | "col" | "row" | "mat"
    data: object = None        # torch tensor (None for scalars)
    coef: float = 1.0          # pending scalar factor (the value itself for scalars)
    trans: bool = False

    @property
    def shape(self):           # logical shape
        if self.kind == "mat":
            r, c = self.data.shape
            return (c, r) if self.trans else (r, c)
        return tuple(self.data.shape)


class _Executor:
    def __init__(self, stream=None):
        import torch
        self.torch = torch
        self.lib = _native.load()
        self.stream = stream or torch.cuda.current_stream()

    def _st(self):
        return ctypes.c_void_p(self.stream.cuda_stream)

    @staticmethod
    def _p(t):
        return ctypes.c_void_p(t.data_ptr())

    def _new(self, *shape):
        return self.torch.empty(*shape, dtype=self.torch.float64, device="cuda")

    # -- primitives -----------------------------------------------------------
    def combine(self, a, ca: float, b, cb: float):
        """ca*a + cb*b elementwise (same-shaped contiguous tensors)."""
        out = self._new(a.shape)
        if ca == 1.0 and cb == 1.0:
            mode = 2
        elif ca == 1.0 and cb == -1.0:
            mode = 3
        else:
            mode = 1
        _native.check(self.lib.bto_prim_axpby_async(ca, self._p(a), cb, self._p(b), self._p(out),
                                                    a.numel(), mode, self._st()))
        return out

    def scaled(self, a, coef: float):
        if coef == 1.0:
            return a
        out = self._new(a.shape)
        _native.check(self.lib.bto_prim_axpby_async(coef, self._p(a), 0.0, None, self._p(out),
                                                    a.numel(), 0, self._st()))
        return out

    def matvec(self, mat: GenericValue, vec) -> object:
        rows, cols = mat.data.shape               # of the stored row-major buffer
        transposed = 1 if mat.trans else 0
        out = self._new(cols if transposed else rows)
        _native.check(self.lib.bto_prim_matvec_async(self._p(mat.data), self._p(vec), self._p(out),
                                                     rows, cols, transposed, self._st()))
        return out

    def dot(self, x, y) -> float:
        out = self._new(1)
        _native.check(self.lib.bto_prim_dot_async(self._p(x), self._p(y), self._p(out), x.numel(),
                                                  self._st()))
        self.stream.synchronize()
        return float(out[0])

    def outer(self, u, v):
        out = self._new(u.numel(), v.numel())
        _native.check(self.lib.bto_prim_outer_async(self._p(u), self._p(v), self._p(out),
                                                    u.numel(), v.numel(), self._st()))
        return out

    # -- expression evaluation --------------------------------------------------
    def transpose(self, v: GenericValue) -> GenericValue:
        if v.kind == "scalar":
            raise KernelSpecError("cannot transpose a scalar")
        if v.kind == "mat":
            return GenericValue("mat", v.data, v.coef, not v.trans)
        return GenericValue("row" if v.kind == "col" else "col", v.data, v.coef)

    def add(self, op: str, a: GenericValue, b: GenericValue) -> GenericValue:
        if a.kind != b.kind:
            raise KernelSpecError(f"cannot combine {a.kind} and {b.kind} with {op!r}")
        sign = 1.0 if op == "+" else -1.0
        if a.kind == "scalar":
            return GenericValue("scalar", coef=a.coef + sign * b.coef)
        if a.shape != b.shape:
            raise KernelSpecError(f"extent mismatch: {a.shape} vs {b.shape}")
        bd = b.data
        if a.kind == "mat" and a.trans != b.trans:          # bring b into a's storage order
            bd = bd.t().contiguous()
        return GenericValue(a.kind, self.combine(a.data, a.coef, bd, sign * b.coef), 1.0,
                            a.trans if a.kind == "mat" else False)

    def mul(self, a: GenericValue, b: GenericValue) -> GenericValue:
        if a.kind == "scalar" or b.kind == "scalar":
            s, v = (a, b) if a.kind == "scalar" else (b, a)
            if v.kind == "scalar":
                return GenericValue("scalar", coef=s.coef * v.coef)
            return GenericValue(v.kind, v.data, s.coef * v.coef, v.trans)
        if a.kind == "row" and b.kind == "col":
            if a.shape != b.shape:
                raise KernelSpecError("dot product extent mismatch")
            return GenericValue("scalar", coef=a.coef * b.coef * self.dot(a.data, b.data))
        if a.kind == "col" and b.kind == "row":
            return GenericValue("mat", self.outer(a.data, b.data), a.coef * b.coef)
        if a.kind == "mat" and b.kind == "col":
            if a.shape[1] != b.shape[0]:
                raise KernelSpecError(f"matrix-vector extent mismatch: {a.shape} x {b.shape}")
            return GenericValue("col", self.matvec(a, b.data), a.coef * b.coef)
        raise KernelSpecError(f"cannot multiply {a.kind} by {b.kind}")

    def evaluate(self, expr, env) -> GenericValue:
        tag = expr[0]
        if tag == "var":
            return env[expr[1]]
        if tag == "t":
            return self.transpose(self.evaluate(expr[1], env))
        left, right = self.evaluate(expr[1], env), self.evaluate(expr[2], env)
        return self.mul(left, right) if tag == "*" else self.add(tag, left, right)

    def materialise(self, v: GenericValue) -> GenericValue:
        if v.kind == "scalar" or v.coef == 1.0:
            return v
        return GenericValue(v.kind, self.scaled(v.data, v.coef), 1.0, v.trans)


def run_generic(graph: TypedSpec, inputs: dict, extents: dict, stream=None) -> dict:
    """Evaluate `graph.spec` on the current CUDA device.

    numpy inputs are copied to the device and the outputs come back as numpy;
    torch CUDA tensors are used in place and the outputs are CUDA tensors.
    Shapes are checked like runtime.run_kernel (ValueError on a mismatch)."""
    import numpy as np
    import torch

    ex = _Executor(stream)
    spec = graph.spec
    on_gpu = any(hasattr(inputs.get(n), "is_cuda") and inputs[n].is_cuda for n, _ in spec.inputs)
    env: dict[str, GenericValue] = {}
    for name, decl in spec.inputs:
        if name not in inputs:
            raise ValueError(f"missing input {name!r}")
        value = inputs[name]
        if decl.kind == "scalar":
            env[name] = GenericValue("scalar", coef=float(value))
            continue
        want = tuple(int(extents[d]) for d in graph.dims[name])
        if tuple(np.shape(value)) != want:
            raise ValueError(f"{name}: expected shape {want}, got {tuple(np.shape(value))}")
        t = value.to("cuda", torch.float64) if hasattr(value, "is_cuda") else _native.to_device(value)
        if decl.kind == "vector":
            env[name] = GenericValue("col" if decl.orientation == "column" else "row", t.contiguous())
        elif decl.orientation == "column":       # column-major operand: store the transpose
            env[name] = GenericValue("mat", t.t().contiguous(), 1.0, True)
        else:
            env[name] = GenericValue("mat", t.contiguous())
    for target, expr in spec.statements:
        env[target] = ex.materialise(ex.evaluate(expr, env))
    outputs = {}
    for name, decl in spec.outputs:
        v = env[name]
        if decl.kind == "scalar":
            if v.kind != "scalar":
                raise KernelSpecError(f"{name!r} declared scalar, computed {v.kind}")
            outputs[name] = float(v.coef)
            continue
        want = tuple(int(extents[d]) for d in graph.dims[name])
        data = v.data
        if v.kind == "mat" and v.trans:
            data = data.t()
        if tuple(data.shape) != want:
            raise ValueError(f"{name}: computed shape {tuple(data.shape)}, declared {want}")
        data = data.contiguous()
        outputs[name] = data if on_gpu else _native.to_host(data)
    ex.stream.synchronize()
    return outputs
