"""Generic (unfused) executor: any valid spec runs on the device."""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import golden_util as G
import np_interp
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import spec as S


def test_numpy_interpreter_matches_reference_interpreter_goldens():
    """Pin tests/np_interp.py against O1 = reference_evaluate for the corpus (CPU)."""
    for name in bto.CORPUS:
        graph = bto.load_graph(name)
        for (m, n, seed) in G.small_cases(name)[:12]:
            ext = {"M": m} if graph.extent_names == ("M",) else {"M": m, "N": n}
            inputs = bto.random_inputs(graph, ext, seed=seed)
            got = np_interp.evaluate(graph.spec, inputs)
            assert G.max_err(got, G.expected(name, f"small/{m}x{n}/s{seed}", "O1")) < 1e-13, name


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
}


def _inputs(typed, ext, seed):
    return bto.gen_inputs(typed, ext, seed=seed)


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(SPECS))
def test_non_corpus_specs_run_unfused(bto_lib, key):
    typed = S.infer_shapes(S.parse_kernel(SPECS[key]))
    kernel = bto.gpu_kernel(typed)
    assert kernel.source.endswith(":generic")
    for (m, n) in [(1, 1), (7, 50), (300, 129), (513, 1026)]:
        ext = {e: (m if e == "M" else n) for e in typed.extent_names}
        inputs = _inputs(typed, ext, seed=m + n)
        want = np_interp.evaluate(typed.spec, inputs)
        tol = 1e-12 * max(1.0, math.log2(max(ext.values())))
        got = bto.run_kernel(bto.library_path(), kernel, typed, inputs, ext)        # numpy in/out
        assert bto.max_rel_error(got, want) <= tol, (key, ext)
        dev = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in inputs.items()}
        got = bto.run_kernel(bto.library_path(), kernel, typed, dev, ext)           # CUDA tensors
        assert all(not isinstance(v, np.ndarray) for v in got.values())
        assert bto.max_rel_error(got, want) <= tol, (key, ext, "device")


@pytest.mark.gpu
def test_generic_path_agrees_with_the_fused_sequences(bto_lib, oracle):
    """Every corpus kernel evaluated by the generic executor matches the oracle, so
    the unfused primitives are held to the same gate as the fused kernels."""
    from paper_1205_1098_b200.generic import run_generic
    for name in bto.CORPUS:
        typed = bto.load_graph(name)
        for (m, n) in [(37, 29), (300, 1026), (1031, 514)]:
            ext = {"M": m * n} if typed.extent_names == ("M",) else {"M": m, "N": n}
            inputs = bto.gen_inputs(typed, ext, seed=3)
            want = oracle.oracle_run(name, inputs, ext, threads=8)
            got = run_generic(typed, inputs, ext)
            tol = 1e-12 * max(1.0, math.log2(max(ext.values())))
            assert bto.max_rel_error(got, want) <= tol, (name, ext)
            for out in {"axpydot": ("z",), "gemver": ("B",), "vadd": ("x",), "waxpby": ("w",)}.get(name, ()):
                assert np.array_equal(got[out], want[out]), (name, out)


@pytest.mark.gpu
def test_generic_shape_errors(bto_lib):
    typed = S.infer_shapes(S.parse_kernel(SPECS["vsub"]))
    kernel = bto.gpu_kernel(typed)
    with pytest.raises(ValueError, match="expected shape"):
        bto.run_kernel(bto.library_path(), kernel, typed, {"a": np.zeros(4), "b": np.zeros(5)}, {"M": 4})
