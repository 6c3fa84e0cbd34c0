"""Call interface of the B200 kernels: the GPU side of `matfuse.runtime`.

Mirrors, name for name, what the reference's callers use on the hot path
(SURVEY.md section 8b):

* `GeneratedKernel`  -- cemit.py:25-31 (here the "source" is a prebuilt CUDA
  sequence inside libbto_b200.so, so `source` only names it);
* `gpu_kernel(graph)`-- stands where `emit_c(contract_arrays(lower(org, g)))`
  stood: returns the kernel handle for a spec, or raises
  UnsupportedKernelError;
* `Toolchain`        -- runtime.py:44-83: `compile()` is a cache lookup that
  returns the shared object's path (building it with nvcc if asked to);
* `run_kernel(binary, kernel, graph, inputs, extents)` -- runtime.py:99-150,
  same arguments, same return value, same ValueError on a shape mismatch.
  numpy inputs are passed as HOST pointers (the library stages them); torch
  CUDA tensors are passed zero-copy and outputs come back as CUDA tensors;
* `random_inputs`, `max_rel_error`, `workdir` -- runtime.py:153-175,194.

`graph` may be this package's TypedSpec or the reference's own DataflowGraph
(both expose .spec.inputs/.outputs and per-name dims), so the reference's
tests can drive this module unchanged.
"""
from __future__ import annotations

import math
import ctypes
import tempfile
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native
from .spec import (KernelSpec, TypedSpec, infer_shapes, load_typed,
                   match_corpus, parse_kernel)

__all__ = [
    "GeneratedKernel", "Toolchain", "ToolchainError", "gpu_kernel",
    "load_graph", "run_kernel", "run_kernel_async", "random_inputs",
    "gen_inputs", "max_rel_error", "workdir", "CHECK_CONFIGS", "BENCH_CONFIGS",
    "SEEDS",
]


class ToolchainError(RuntimeError):
    """Same role as runtime.py:29 -- the kernel could not be built or run."""


@dataclass(frozen=True)
class GeneratedKernel:
    source: str                               # "libbto_b200:<kernel>"
    kernel_name: str                          # C symbol (spec.name.lower())
    params: tuple[tuple[str, str], ...]       # (C declaration, logical name)
    organism_key: str                         # fused sequence description
    threads: tuple[int, ...] = ()             # unused on the GPU (grid is planned)


#: how each corpus kernel is fused on the GPU (shown as organism_key)
_SEQUENCES = {
    "axpydot": "gpu{k: 1 2 3 | grid-reduce}",
    "vadd": "gpu{k: 1 2}",
    "waxpby": "gpu{k: 1 2 3}",
    "bicgk": "gpu{strip(j) rows(i): 1 2 | join q,s}",
    # one pass: a cluster holds a row panel in shared memory / registers between the two products
    "atax": "gpu{cluster rows(i): {j: 1}{j: 2} | join y}",
    "batax": "gpu{cluster rows(i): {j: 1}{j: 2} | join,scale y}",
    "gesummv": "gpu{strip(j) rows(i): 1 3 | join 2 4 5}",
    "dgemv": "gpu{strip(j) rows(i): 1 | join 2 3 4}",
    "gemver": "gpu{strip(j) rows(i): 1 2 3 4 5 | join 6 7}{strip(j) rows(i): 8 | join 9}",
    "dgemvt": "gpu{strip(j) rows(i): 1 | join 2 3}{strip(j) rows(i): 4 | join 5}",
}


def _is_reference_graph(graph) -> bool:
    """matfuse's DataflowGraph (graph.py): carries `.data` (name -> typed node) and `.spec`."""
    return hasattr(graph, "data") and hasattr(graph, "spec") and not isinstance(graph, TypedSpec)


def _spec_from_reference(graph) -> KernelSpec:
    """The reference's parsed spec (lang.py dataclasses) as this package's KernelSpec."""
    from .spec import Decl
    spec = graph.spec
    return KernelSpec(
        spec.name,
        tuple((n, Decl(d.kind, d.orientation)) for n, d in spec.inputs),
        tuple((n, Decl(d.kind, d.orientation)) for n, d in spec.outputs),
        tuple((s.target, _convert_expr(s.value)) for s in spec.statements))


def _as_typed(graph) -> TypedSpec:
    if isinstance(graph, TypedSpec):
        return graph
    if isinstance(graph, KernelSpec):
        return infer_shapes(graph)
    if isinstance(graph, str):
        return infer_shapes(parse_kernel(graph))
    if _is_reference_graph(graph):
        return infer_shapes(_spec_from_reference(graph))
    raise TypeError(f"cannot interpret {type(graph).__name__} as a kernel spec")


def load_graph(name: str) -> TypedSpec:
    """Corpus kernel by name (the reference's corpus.load_graph, corpus.py:46)."""
    return load_typed(name)


def _c_params(inputs, outputs, extent_names) -> tuple[tuple[str, str], ...]:
    out = []
    for name, decl in inputs:
        out.append((f"double {name}" if decl.kind == "scalar"
                    else f"const double *{name}", name))
    for name, decl in outputs:
        out.append((f"double *{name}", name))
    out += [(f"long {e}", e) for e in extent_names]
    return tuple(out)


def gpu_kernel(graph, allow_generic: bool = True, allow_emitted: bool = True) -> GeneratedKernel:
    """The kernel handle for `graph`'s spec: the hand-written fused sm_100a
    sequence when the spec is one of the corpus structures (row-major, or all
    column-major); otherwise -- mixed orientations, kernels outside the corpus --
    FUSED CUDA emitted for the organism the reference's search picks under the
    GPU cost model (`cuemit.emitted_kernel_for`: needs the reference and nvcc,
    i.e. the drop-in setting; the reference emits fused C for any spec,
    cemit.py:54-72); failing that (unless `allow_generic=False`, which raises
    UnsupportedKernelError) the generic unfused executor of generic.py."""
    from .spec import UnsupportedKernelError
    typed = _as_typed(graph)          # (the reference's own DataflowGraph is converted)
    spec = typed.spec
    params = _c_params(spec.inputs, spec.outputs, typed.extent_names)
    try:
        name = match_corpus(spec)
    except UnsupportedKernelError:
        from .colmajor import column_major_variant
        cm = column_major_variant(spec)
        if cm is not None:      # a corpus kernel on column-major matrices: fused, roles swapped
            return GeneratedKernel(
                source=f"libbto_b200:colmajor:{cm}", kernel_name=spec.name.lower(), params=params,
                organism_key="colmajor " + _SEQUENCES[cm])
        if allow_emitted:
            from .cuemit import emitted_kernel_for
            try:
                emitted = emitted_kernel_for(graph if _is_reference_graph(graph) else typed)
            except ToolchainError:
                emitted = None
            if emitted is not None:
                return emitted
        if not allow_generic:
            raise
        return GeneratedKernel(
            source="libbto_b200:generic", kernel_name=spec.name.lower(), params=params,
            organism_key="gpu-unfused{" + " ".join(str(i + 1) for i in range(len(spec.statements))) + "}")
    return GeneratedKernel(
        source=f"libbto_b200:{name}", kernel_name=name, params=params,
        organism_key=_SEQUENCES[name])


def _convert_expr(e):
    """matfuse.lang AST (Var/Transpose/BinOp dataclasses) -> our tuples."""
    cls = type(e).__name__
    if cls == "Var":
        return ("var", e.name)
    if cls == "Transpose":
        return ("t", _convert_expr(e.operand))
    return (e.op, _convert_expr(e.left), _convert_expr(e.right))


@dataclass
class Toolchain:
    """`compile()` returns the prebuilt library; `rebuild=True` runs nvcc first.

    The reference compiles generated C per organism (runtime.py:70-83); here
    the kernels are hand-written and prebuilt, so compiling is a cache lookup.
    """
    rebuild: bool = False

    @property
    def available(self) -> bool:
        return _native.library_path().exists()

    def compile(self, source: str = "", workdir=None, name: str = "kernel",
                shared: bool = True) -> Path:
        if not shared:
            raise ToolchainError(
                "standalone timing binaries are not produced on the GPU path; "
                "time with paper_1205_1098_b200.cost.GpuEmpiricalTimer")
        if self.rebuild:
            from .build import build_library
            try:
                build_library()
            except Exception as exc:  # nvcc failure
                raise ToolchainError(f"compile failed: {exc}") from exc
        path = _native.library_path()
        if not path.exists():
            raise ToolchainError(f"compile failed: {path} does not exist")
        return path


def _dims(graph, name: str) -> tuple[str, ...]:
    if hasattr(graph, "dims") and not hasattr(graph, "data"):
        return tuple(graph.dims[name])
    return tuple(graph.data[name].dims)


def _is_cuda_tensor(value) -> bool:
    return hasattr(value, "is_cuda") and bool(value.is_cuda)


def _marshal(binary, kernel: GeneratedKernel, graph, inputs: dict, extents: dict):
    """Build the C argument list.  Returns (fn, args, out_bufs, keepalive, on_gpu)."""
    lib = _native.load()
    if Path(binary).resolve() != _native.library_path().resolve():
        raise ToolchainError(f"{binary} is not the loaded kernel library")
    spec = graph.spec
    on_gpu = any(_is_cuda_tensor(inputs.get(n)) for n, _ in spec.inputs)
    if on_gpu:
        import torch
    args, keep, out_bufs = [], [], {}
    for name, decl in spec.inputs:
        if name not in inputs:
            raise ValueError(f"missing input {name!r}")
        value = inputs[name]
        if decl.kind == "scalar":
            args.append(ctypes.c_double(float(value)))
            continue
        want = tuple(int(extents[d]) for d in _dims(graph, name))
        if _is_cuda_tensor(value):
            if tuple(value.shape) != want:
                raise ValueError(f"{name}: expected shape {want}, got {tuple(value.shape)}")
            if value.dtype != torch.float64:
                raise ValueError(f"{name}: expected float64, got {value.dtype}")
            flat = value.contiguous()
            keep.append(flat)
            args.append(ctypes.c_void_p(flat.data_ptr()))
        else:
            if on_gpu:
                raise ValueError(f"{name}: mixing CUDA tensors and host arrays")
            arr = np.asarray(value, dtype=np.float64)
            if arr.shape != want:
                raise ValueError(f"{name}: expected shape {want}, got {arr.shape}")
            flat = np.ascontiguousarray(arr.ravel(order="C"))
            keep.append(flat)
            args.append(ctypes.c_void_p(flat.ctypes.data))
    for name, decl in spec.outputs:
        size = 1
        for d in _dims(graph, name):
            size *= int(extents[d])
        if on_gpu:
            # NaN prefill, as runtime.py:108,130: an unwritten element is loud
            buf = torch.full((size,), float("nan"), dtype=torch.float64,
                             device=keep[0].device if keep else "cuda")
            args.append(ctypes.c_void_p(buf.data_ptr()))
        else:
            buf = _native.filled(size, np.nan) if size >= (1 << 20) else np.full(size, np.nan, dtype=np.float64)
            args.append(ctypes.c_void_p(buf.ctypes.data))
        out_bufs[name] = buf
        keep.append(buf)
    for ext in graph.extent_names:
        args.append(ctypes.c_long(int(extents[ext])))
    return lib, args, out_bufs, keep, on_gpu


def _unpack(graph, extents: dict, out_bufs: dict, on_gpu: bool) -> dict:
    outputs = {}
    for name, decl in graph.spec.outputs:
        buf = out_bufs[name]
        if decl.kind == "scalar":
            outputs[name] = float(buf[0])
        else:
            shape = tuple(int(extents[d]) for d in _dims(graph, name))
            outputs[name] = buf.reshape(shape)
    return outputs


def run_kernel(binary, kernel: GeneratedKernel, graph, inputs: dict,
               extents: dict) -> dict:
    """Run the kernel on `inputs`; returns the outputs dict (runtime.py:99-150).

    numpy in -> numpy out (host buffers cross PCIe inside the call);
    torch CUDA tensors in -> CUDA tensors out, synchronised before returning.
    """
    if kernel.source.endswith(":generic"):
        from .generic import run_generic
        return run_generic(_as_typed(graph), inputs, extents)
    if kernel.source.startswith("emitted:"):
        from .cuemit import emitted_entry, run_emitted
        path, emitted, ir = emitted_entry(kernel.source)
        return run_emitted(path, emitted, ir, inputs, extents)
    if ":colmajor:" in kernel.source:
        from .colmajor import run_colmajor
        return run_colmajor(kernel.source.rsplit(":", 1)[1], _as_typed(graph), inputs, extents)
    lib, args, out_bufs, keep, on_gpu = _marshal(binary, kernel, graph, inputs, extents)
    fn = getattr(lib, kernel.kernel_name)
    if on_gpu:
        import torch
        stream = torch.cuda.current_stream()
        afn = getattr(lib, f"bto_{kernel.kernel_name}_async")
        _native.check(afn(*args, ctypes.c_void_p(stream.cuda_stream)))
        stream.synchronize()
    else:
        fn(*args)
        _native.check()
    del keep
    return _unpack(graph, extents, out_bufs, on_gpu)


def run_kernel_async(kernel: GeneratedKernel, graph, inputs: dict, extents: dict,
                     outputs: dict, stream=None) -> None:
    """Enqueue the kernel on `stream` writing into caller-owned CUDA tensors
    (`outputs` maps every output name to a float64 CUDA tensor; a scalar output
    is a 1-element tensor).  No allocation, no synchronisation: this is what
    the timing loop and the sharded runtime call."""
    import torch
    lib = _native.load()
    spec = graph.spec
    args = []
    for name, decl in spec.inputs:
        value = inputs[name]
        if decl.kind == "scalar":
            args.append(ctypes.c_double(float(value)))
        else:
            want = tuple(int(extents[d]) for d in _dims(graph, name))
            if tuple(value.shape) != want or value.dtype != torch.float64 \
                    or not value.is_cuda or not value.is_contiguous():
                raise ValueError(f"{name}: expected contiguous float64 CUDA tensor of shape {want}")
            args.append(ctypes.c_void_p(value.data_ptr()))
    for name, decl in spec.outputs:
        buf = outputs[name]
        size = 1
        for d in _dims(graph, name):
            size *= int(extents[d])
        if buf.numel() != size or buf.dtype != torch.float64 or not buf.is_cuda \
                or not buf.is_contiguous():
            raise ValueError(f"{name}: expected contiguous float64 CUDA tensor of {size} elements")
        args.append(ctypes.c_void_p(buf.data_ptr()))
    for ext in graph.extent_names:
        args.append(ctypes.c_long(int(extents[ext])))
    if stream is None:
        stream = torch.cuda.current_stream()
    afn = getattr(lib, f"bto_{kernel.kernel_name}_async")
    _native.check(afn(*args, ctypes.c_void_p(stream.cuda_stream)))


def random_inputs(graph, extents: dict, seed: int = 0) -> dict:
    """The reference's validation inputs (runtime.py:153-164): arrays U[-1,1),
    scalars U[0.1,1), drawn in declaration order from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    inputs = {}
    for name, decl in graph.spec.inputs:
        if decl.kind == "scalar":
            inputs[name] = float(rng.uniform(0.1, 1.0))
        else:
            shape = tuple(int(extents[d]) for d in _dims(graph, name))
            inputs[name] = rng.uniform(-1.0, 1.0, size=shape)
    return inputs


def gen_inputs(graph, extents: dict, seed: int = 0) -> dict:
    """BASELINE.json's inputs: as random_inputs but the
    scalars are U[-1,1) too."""
    rng = np.random.default_rng(seed)
    inputs = {}
    for name, decl in graph.spec.inputs:
        if decl.kind == "scalar":
            inputs[name] = float(rng.uniform(-1.0, 1.0))
        else:
            shape = tuple(int(extents[d]) for d in _dims(graph, name))
            inputs[name] = rng.uniform(-1.0, 1.0, size=shape)
    return inputs


def max_rel_error(got: dict, want: dict) -> float:
    """The reference's error metric (runtime.py:167-175): max over outputs of
    |g - e| / max(|e|, 1).  Unlike the reference's (where `max(0.0, nan)` is 0.0) a
    non-finite element anywhere -- an output the kernel left at its NaN prefill --
    yields `inf`: this function is the validator of the product path."""
    worst = 0.0
    for name, expected in want.items():
        g = got[name]
        if _is_cuda_tensor(g):
            g = g.cpu().numpy()
        g = np.asarray(g, dtype=np.float64)
        e = np.asarray(expected, dtype=np.float64)
        if e.size == 0:
            continue
        if g.shape != e.shape:
            if g.size != e.size:
                return math.inf
            g = g.reshape(e.shape)
        err = float(np.max(np.abs(g - e) / np.maximum(np.abs(e), 1.0)))
        if not math.isfinite(err):
            return math.inf
        worst = max(worst, err)
    return worst


def workdir() -> Path:
    return Path(tempfile.mkdtemp(prefix="bto-b200-"))


#: BASELINE.json configs: seeds, CPU-check extents and GPU bench extents
SEEDS = {"axpydot": 0, "bicgk": 1, "atax": 2, "gesummv": 3, "gemver": 4}
CHECK_CONFIGS = {
    "axpydot": {"M": 1 << 20},
    "bicgk": {"M": 2048, "N": 2048},
    "atax": {"M": 2048, "N": 1024},
    "gesummv": {"M": 2048, "N": 2048},
    "gemver": {"M": 2048, "N": 2048},
}
BENCH_CONFIGS = {
    "axpydot": {"M": 1 << 27},
    "bicgk": {"M": 32768, "N": 32768},
    "atax": {"M": 32768, "N": 32768},
    "gesummv": {"M": 24576, "N": 24576},
    "gemver": {"M": 32768, "N": 32768},
}
