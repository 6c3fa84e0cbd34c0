"""Generic (unfused) executor: any valid spec runs on the device."""
from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np
import pytest
import torch

import golden_util as G
import np_interp
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import _native
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


from noncorpus_specs import EXTENTS, SPECS  # noqa: E402

def _inputs(typed, ext, seed):
    return bto.gen_inputs(typed, ext, seed=seed)


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(SPECS))
def test_non_corpus_specs_run_unfused(bto_lib, key):
    typed = S.infer_shapes(S.parse_kernel(SPECS[key]))
    kernel = bto.gpu_kernel(typed, allow_emitted=False)
    assert kernel.source.endswith(":generic")
    for (m, n) in EXTENTS:
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


def test_format_kernel_round_trips():
    for text in SPECS.values():
        spec = S.parse_kernel(text)
        assert S.parse_kernel(S.format_kernel(spec)) == spec
    for name in bto.CORPUS:
        spec = S.load_spec(name)
        assert S.parse_kernel(S.format_kernel(spec)) == spec


def _reference_importable() -> bool:
    import importlib.util
    import sys
    ref = "/root/reference/pkg/src"
    if importlib.util.find_spec("matfuse") is None and __import__("os").path.isdir(ref):
        sys.path.insert(0, ref)
        sys.dont_write_bytecode = True
    return importlib.util.find_spec("matfuse") is not None


def test_specs_outside_the_hand_written_set_get_fused_emitted_code(tmp_path, monkeypatch):
    """Where the reference and nvcc are present (the drop-in setting), `gpu_kernel` answers a
    mixed-orientation or non-corpus spec with FUSED CUDA emitted for the organism the reference's
    search picks under the GPU cost model -- not with the statement-by-statement executor -- and
    the organism is the one stored in tests/golden/noncorpus.json (what the GPU box runs)."""
    from paper_1205_1098_b200 import cuemit
    if not _reference_importable() or not cuemit.NvccToolchain().available:
        pytest.skip("needs the reference (matfuse) and nvcc")
    monkeypatch.setenv("BTO_NVCC_CACHE", str(tmp_path / "cache"))
    stored = json.loads((Path(__file__).parent / "golden" / "noncorpus.json").read_text())
    for key in ("gemver_mixed", "mixed", "dotscale"):
        typed = S.infer_shapes(S.parse_kernel(SPECS[key]))
        kernel = bto.gpu_kernel(typed)
        assert kernel.source.startswith("emitted:") and Path(kernel.source[len("emitted:"):]).exists()
        assert kernel.kernel_name == typed.spec.name.lower()
        assert kernel.organism_key == stored[key]["ir"]["organism"]
        assert [n for _, n in kernel.params] == [n for n, _ in typed.spec.inputs + typed.spec.outputs] + list(typed.extent_names)
        _, emitted, ir = cuemit.emitted_entry(kernel.source)
        assert ir == stored[key]["ir"] and "_region0" in emitted.source
    # the reference's own DataflowGraph is accepted in place of a TypedSpec: corpus kernels get the
    # hand-written sequence, anything else the same emitted code
    import matfuse
    from matfuse.corpus import load_graph as ref_load
    from matfuse.graph import build_dataflow, infer_types
    assert bto.gpu_kernel(ref_load("gemver")).source == "libbto_b200:gemver"
    ref_mixed = infer_types(build_dataflow(matfuse.parse_kernel(S.format_kernel(S.parse_kernel(SPECS["mixed"])))))
    k = bto.gpu_kernel(ref_mixed)
    assert k.source.startswith("emitted:") and k.organism_key == stored["mixed"]["ir"]["organism"]
    assert bto.gpu_kernel(ref_mixed, allow_emitted=False).source == "libbto_b200:generic"
    # without the toolchain the unfused executor answers
    monkeypatch.setattr(cuemit.NvccToolchain, "available", property(lambda self: False))
    assert bto.gpu_kernel(S.infer_shapes(S.parse_kernel(SPECS["mixed"]))).source.endswith(":generic")


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(SPECS))
def test_emitted_fused_code_for_specs_outside_the_hand_written_set(bto_lib, tmp_path, key):
    """The stored organisms of tests/golden/noncorpus.json (chosen by the reference's search under
    the GPU cost model, tests/golden/make_noncorpus.py) emitted, compiled and run through
    `run_kernel`: results equal the reference interpreter's stored O1 values and the numpy
    restatement, host and device operands; matrix outputs with mixed orientations included."""
    from paper_1205_1098_b200 import cuemit
    stored = json.loads((Path(__file__).parent / "golden" / "noncorpus.json").read_text())[key]
    typed = S.infer_shapes(S.parse_kernel(stored["spec"]))
    kernel = cuemit.emitted_kernel_for(typed, toolchain=cuemit.NvccToolchain(cache_dir=str(tmp_path)), ir=stored["ir"])
    assert kernel is not None and kernel.source.startswith("emitted:")
    for case in stored["cases"]:
        ext = case["ext"]
        inputs = bto.random_inputs(typed, ext, seed=case["seed"])
        want = np_interp.evaluate(typed.spec, inputs)
        tol = 1e-12 * max(1.0, math.log2(max(ext.values())))
        _native.poison_shared_memory()
        got = bto.run_kernel(bto.library_path(), kernel, typed, inputs, ext)
        assert bto.max_rel_error(got, want) <= tol, (key, ext)
        for name, head in case["out"].items():          # the reference's own O1 values
            mine = np.asarray(got[name], dtype=np.float64).ravel()[:64] if not isinstance(head, float) else got[name]
            assert np.allclose(mine, head, rtol=1e-11, atol=1e-11), (key, ext, name)
            assert math.isclose(float(np.sum(np.asarray(got[name]))), case["sum"][name], rel_tol=1e-9, abs_tol=1e-8)
        dev = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in inputs.items()}
        got = bto.run_kernel(bto.library_path(), kernel, typed, dev, ext)
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
