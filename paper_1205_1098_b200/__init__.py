"""paper_1205_1098_b200 -- B200-native execution of the BTO fused BLAS-1/BLAS-2
sequences (AXPYDOT, BiCGK, ATAX, GESUMMV, GEMVER, ...), a drop-in for the
generated-C path of the reference `matfuse` package.

Public names follow the reference's (`matfuse/__init__.py:10-34`) where the
hot path has an equivalent.  Importing the package does not load the CUDA
library; the first kernel call does, and fails loudly if it is missing.
"""
from .spec import (CORPUS, HOT_PATH, KernelSpec, KernelSpecError,
                   KernelSyntaxError, TypedSpec, UnsupportedKernelError,
                   infer_shapes, load_spec, load_typed, parse_kernel)
from .runtime import (BENCH_CONFIGS, CHECK_CONFIGS, SEEDS, GeneratedKernel,
                      Toolchain, ToolchainError, gen_inputs, gpu_kernel,
                      load_graph, max_rel_error, random_inputs, run_kernel,
                      run_kernel_async, workdir)
from ._native import BtoError, NativeLibraryMissing, library_path
from .cost import (AnalyticGpuCost, CostReport, GpuEmpiricalTimer, GpuMachineModel, GpuVariant,
                   cached, estimate_cost)
from .search import SearchConfig, SearchResult, run_strategy

__version__ = "0.1.0"

__all__ = [
    "CORPUS", "HOT_PATH", "KernelSpec", "KernelSpecError", "KernelSyntaxError",
    "TypedSpec", "UnsupportedKernelError", "infer_shapes", "load_spec",
    "load_typed", "parse_kernel",
    "BENCH_CONFIGS", "CHECK_CONFIGS", "SEEDS", "GeneratedKernel", "Toolchain",
    "ToolchainError", "gen_inputs", "gpu_kernel", "load_graph", "max_rel_error",
    "random_inputs", "run_kernel", "run_kernel_async", "workdir",
    "BtoError", "NativeLibraryMissing", "library_path",
    "AnalyticGpuCost", "CostReport", "GpuEmpiricalTimer", "GpuMachineModel", "GpuVariant",
    "cached", "estimate_cost", "SearchConfig", "SearchResult", "run_strategy",
]
