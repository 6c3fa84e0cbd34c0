"""Kernel-spec front end of the drop-in boundary (no GPU)."""
from __future__ import annotations

import pytest

import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import spec as S

BATAX_SRC = """
BATAX
in:
    x : vector(column), beta : scalar,
    A : matrix(row)
out:
    y : vector(column)
{
    y = beta * A' * (A * x)
}
"""


def test_parse_multiline_source_and_match():
    spec = S.parse_kernel(BATAX_SRC)
    assert spec.name == "BATAX"
    assert [n for n, _ in spec.inputs] == ["x", "beta", "A"]
    assert S.match_corpus(spec) == "batax"


def test_c_signature_order_follows_declaration_order():
    # cemit.py:225-241: inputs, outputs, then sorted extents
    t = bto.load_graph("gemver")
    assert [n for n, _ in t.params()] == [
        "A", "u1", "v1", "u2", "v2", "alpha", "beta", "y", "z", "B", "x", "w", "M", "N"]
    t = bto.load_graph("axpydot")
    assert [n for n, _ in t.params()] == ["w", "v", "u", "alpha", "z", "beta", "M"]
    assert dict(t.params())["beta"] == "scalar_out"


def test_extent_naming():
    # graph.py:459-501: matrix rows M, columns N; vector-only kernels use M
    t = bto.load_graph("bicgk")
    assert t.dims == {"A": ("M", "N"), "p": ("N",), "r": ("M",), "q": ("M",), "s": ("N",)}
    assert bto.load_graph("atax").dims["y"] == ("N",)
    assert bto.load_graph("gesummv").dims["y"] == ("M",)
    assert bto.load_graph("vadd").extent_names == ("M",)


def test_renamed_spec_still_matches():
    text = ("MYKERNEL in: Q : matrix(row), a : vector(column), b : vector(column) "
            "out: c : vector(column), d : vector(column) { c = Q * a  d = Q' * b }")
    assert S.match_corpus(S.parse_kernel(text)) == "bicgk"


def test_unknown_structure_gets_the_generic_executor_or_a_loud_error():
    text = "T in: a : vector(column), b : vector(column) out: c : vector(column) { c = a - b }"
    typed = S.infer_shapes(S.parse_kernel(text))
    with pytest.raises(S.UnsupportedKernelError):
        bto.gpu_kernel(typed, allow_generic=False, allow_emitted=False)
    k = bto.gpu_kernel(typed, allow_emitted=False)      # (with the reference + nvcc: fused emitted code)
    assert k.source == "libbto_b200:generic" and k.kernel_name == "t"
    assert k.organism_key == "gpu-unfused{1}"


def test_declaration_order_matters():
    # same algebra as DGEMV but another argument order -> another C signature
    text = ("D in: A : matrix(row), alpha : scalar, x : vector(column), beta : scalar, "
            "y : vector(column) out: z : vector(column) { z = alpha * A * x + beta * y }")
    with pytest.raises(S.UnsupportedKernelError):
        S.match_corpus(S.parse_kernel(text))


@pytest.mark.parametrize("text, exc", [
    ("K in: a : scalar out: b : scalar { b = c }", S.KernelSpecError),
    ("K in: a : scalar out: b : scalar { a = a }", S.KernelSpecError),
    ("K in: a : scalar out: b : scalar { }", S.KernelSpecError),
    ("K in: a : scalar, a : scalar out: b : scalar { b = a }", S.KernelSpecError),
    ("K in: a : vector(diag) out: b : scalar { b = a }", S.KernelSyntaxError),
    ("K in: a : scalar out: b : scalar { b = a } junk", S.KernelSyntaxError),
    ("K in: a : scalar out: b : scalar { b = a + }", S.KernelSyntaxError),
])
def test_malformed_specs(text, exc):
    with pytest.raises(exc):
        S.parse_kernel(text)


def test_syntax_error_carries_position():
    with pytest.raises(S.KernelSyntaxError) as info:
        S.parse_kernel("K in: a : scalar\nout: b : scalar { b = a $ }")
    assert info.value.line == 2


def test_shape_errors():
    with pytest.raises(S.KernelSpecError):   # rows == columns forced (graph.py:472-476)
        S.infer_shapes(S.parse_kernel(
            "K in: A : matrix(row), x : vector(column) out: y : vector(column) { y = A * (A * x) }"))
    with pytest.raises(S.KernelSpecError):
        S.infer_shapes(S.parse_kernel(
            "K in: A : matrix(row), x : vector(column) out: y : vector(column) { y = A + x }"))


def test_precedence_and_associativity():
    spec = S.parse_kernel("K in: a : scalar, b : scalar, c : scalar out: d : scalar "
                          "{ d = a - b - c * a }")
    _, expr = spec.statements[0]
    assert expr == ("-", ("-", ("var", "a"), ("var", "b")), ("*", ("var", "c"), ("var", "a")))


def test_generated_kernel_handle():
    g = bto.load_graph("gesummv")
    k = bto.gpu_kernel(g)
    assert k.kernel_name == "gesummv"
    assert [n for _, n in k.params] == ["alpha", "beta", "A", "B", "x", "y", "M", "N"]
    assert k.params[0][0] == "double alpha" and k.params[2][0] == "const double *A"


def test_column_major_variants_of_the_corpus_are_recognised():
    """All matrices `matrix(column)` -> the fused column-major mapping (colmajor.py);
    mixed orientations and non-corpus structures are left to the generic executor."""
    from paper_1205_1098_b200 import spec as S
    from paper_1205_1098_b200.colmajor import COLMAJOR_SEQUENCES, column_major_variant
    for name in S.CORPUS:
        text = S.CORPUS[name]
        assert column_major_variant(S.parse_kernel(text)) is None              # row-major: not ours
        col = S.parse_kernel(text.replace("matrix(row)", "matrix(column)"))
        assert column_major_variant(col) == (name if name in COLMAJOR_SEQUENCES else None)
    mixed = S.parse_kernel(S.CORPUS["gesummv"].replace("A : matrix(row)", "A : matrix(column)"))
    assert column_major_variant(mixed) is None
    other = S.parse_kernel("K in: A : matrix(column), x : vector(column) out: y : vector(column) "
                           "{ y = A * x }")
    assert column_major_variant(other) is None
    # gpu_kernel: fused handle with the caller's kernel name and the corpus argument order
    import paper_1205_1098_b200 as bto
    g = S.infer_shapes(S.parse_kernel(S.CORPUS["gemver"].replace("matrix(row)", "matrix(column)")))
    k = bto.gpu_kernel(g, allow_generic=False)
    assert k.source == "libbto_b200:colmajor:gemver" and k.organism_key.startswith("colmajor ")
    assert [n for _, n in k.params][:3] == ["A", "u1", "v1"]
