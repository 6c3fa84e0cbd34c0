"""The C-ABI shared library: loads, exports what include/bto_b200.h declares,
and fails loudly (no CPU fallback) when there is no device.  No GPU needed."""
from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import _native

REPO = Path(__file__).resolve().parent.parent
HEADER = (REPO / "include" / "bto_b200.h").read_text()


def declared_functions() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?(?:unsigned\s+)?(?:void|int|long\s+long|long|double|char)\s*\*?\s*(\w+)\s*\(",
                       text, flags=re.M)
    return sorted(set(names))


def test_library_is_built_in_tree():
    assert _native.library_path().exists(), "run python -m paper_1205_1098_b200.build"
    assert _native.library_path().parent == REPO / "paper_1205_1098_b200"


def test_exports_every_declared_symbol():
    lib = _native.load()
    names = declared_functions()
    assert len(names) >= 35
    for name in names:
        assert hasattr(lib, name), f"{name} declared in bto_b200.h but not exported"
    assert set(_native.EXPORTED) == set(names)
    assert lib.bto_abi_version() == 2


def test_reference_symbol_names_and_signatures():
    # the ten symbols the reference's run_kernel would look up (cemit.py:261)
    for name, sig in _native.SIGNATURES.items():
        typed = bto.load_graph(name)
        letters = "".join({"in": "p", "out": "p", "scalar_out": "p", "scalar": "d",
                           "extent": "l"}[cls] for _, cls in typed.params())
        assert letters == sig, name


def test_bytes_min_formulas():
    # SURVEY.md section 8d figures at the bench configs
    assert _native.bytes_min("axpydot", 1 << 27) == 4294967296
    assert _native.bytes_min("bicgk", 32768, 32768) == 8590983168
    assert _native.bytes_min("atax", 32768, 32768) == 8590458880
    assert _native.bytes_min("gesummv", 24576, 24576) == 9664069632
    assert _native.bytes_min("gemver", 32768, 32768) == 25772163072
    with pytest.raises(KeyError):
        _native.bytes_min("nope", 1, 1)


def test_tuning_keys_are_validated():
    assert _native.get_tuning("mv_rows") in (0, 8, 16)
    assert _native.get_tuning("no_such_key") == -1
    with pytest.raises(_native.BtoError):
        _native.set_tuning(mv_rows=5)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_no_device_is_an_error_not_a_fallback():
    g = bto.load_graph("axpydot")
    inputs = bto.gen_inputs(g, {"M": 8}, seed=0)
    with pytest.raises(_native.BtoError) as info:
        bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, inputs, {"M": 8})
    assert info.value.code in (1, 3)


def test_shape_mismatch_is_a_value_error():
    # runtime.py:89-90
    g = bto.load_graph("bicgk")
    inputs = bto.gen_inputs(g, {"M": 4, "N": 4}, seed=0)
    inputs["p"] = np.zeros(5)
    with pytest.raises(ValueError, match="expected shape"):
        bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, inputs, {"M": 4, "N": 4})


def test_product_code_never_touches_the_oracle():
    for path in (REPO / "paper_1205_1098_b200").rglob("*"):
        if path.suffix in (".py", ".cu", ".cuh", ".h"):
            text = path.read_text()
            assert "oracle_lib" not in text and "libbto_oracle" not in text, path
            assert "/root/reference" not in text, path


def test_host_fill_needs_no_gpu():
    """bto_fill_host (the parallel NaN prefill of large outputs) is pure host code."""
    import numpy as np
    from paper_1205_1098_b200 import _native
    for size, value in ((1, 2.5), (1000, -0.0), ((3 << 20) + 3, float("nan")), (5 << 20, 1e300)):
        out = _native.filled(size, value)
        assert out.shape == (size,) and out.dtype == np.float64
        want = np.full(size, value)
        assert np.array_equal(out.view(np.uint64), want.view(np.uint64))
