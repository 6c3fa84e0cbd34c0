"""ctypes binding of libbto_b200.so (include/bto_b200.h).

The library is built in-tree by `paper_1205_1098_b200.build` (nvcc, sm_100a) and
loaded from the package directory.  There is no fallback: if the shared
object is missing or a call fails, this module raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_long, c_void_p
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_NAME = "libbto_b200.so"

_D = c_double
_P = c_void_p          # device or host `double*`, passed as an integer address
_L = c_long
_S = c_void_p          # cudaStream_t


class BtoError(RuntimeError):
    """A libbto_b200 call failed (CUDA error, bad argument, no device)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"libbto_b200 error {code}: {message}")
        self.code = code


class NativeLibraryMissing(ImportError):
    pass


# argument lists of the section-1 symbols, in C order: "p" pointer, "d" double,
# "l" long.  The *_async variants append a stream.
SIGNATURES = {
    "axpydot": "pppdppl",
    "bicgk": "pppppll",
    "atax": "pppll",
    "gesummv": "ddppppll",
    "gemver": "pppppddpppppll",
    "vadd": "ppppl",
    "waxpby": "dpdppl",
    "dgemv": "dppdppll",
    "dgemvt": "ddpppppll",
    "batax": "pdppll",
}
_CT = {"p": _P, "d": _D, "l": _L}

#: every symbol include/bto_b200.h declares (tests check the library exports them)
EXPORTED = tuple(SIGNATURES) + tuple(f"bto_{k}_async" for k in SIGNATURES) + (
    "bto_gemver_pass1_async", "bto_gemver_xupdate_async", "bto_gemver_pass2_async",
    "bto_exchange_init", "bto_exchange_shutdown", "bto_exchange_flag_bytes", "bto_exchange_status",
    "bto_axpydot_sharded_async", "bto_bicgk_sharded_async", "bto_atax_sharded_async",
    "bto_gemver_sharded_async",
    "bto_prim_matvec_async", "bto_prim_axpby_async", "bto_prim_outer_async", "bto_prim_dot_async",
    "bto_colsum_axpz_async", "bto_rank2_rowdot_async",
    "bto_last_error", "bto_last_error_string", "bto_clear_error",
    "bto_abi_version", "bto_set_stream", "bto_set_tuning", "bto_get_tuning",
    "bto_kernel_launches", "bto_last_launch_signature", "bto_last_launch_plan", "bto_bytes_min", "bto_device_info",
    "bto_workspace_bytes", "bto_release_workspace", "bto_reserve_workspace", "bto_copy_to_device", "bto_copy_to_host", "bto_fill_host",
    "bto_debug_poison_shared_memory", "bto_debug_poison_workspace", "bto_debug_poison_all",
)

_lib = None


def library_path() -> Path:
    override = os.environ.get("BTO_B200_LIB")
    return Path(override) if override else PKG_DIR / LIB_NAME


def load() -> ctypes.CDLL:
    """dlopen the library once and declare every prototype."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not path.exists():
        raise NativeLibraryMissing(
            f"{path} not found: build it with `python -m paper_1205_1098_b200.build` "
            "(nvcc, sm_100a); there is no CPU fallback")
    lib = ctypes.CDLL(str(path))
    for name, sig in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = None
        fn.argtypes = [_CT[ch] for ch in sig]
        afn = getattr(lib, f"bto_{name}_async")
        afn.restype = c_int
        afn.argtypes = [_CT[ch] for ch in sig] + [_S]
    lib.bto_gemver_pass1_async.restype = c_int
    lib.bto_gemver_pass1_async.argtypes = [_P] * 8 + [_L, _L, _S]
    lib.bto_gemver_xupdate_async.restype = c_int
    lib.bto_gemver_xupdate_async.argtypes = [_P, _D, _P, _P, _L, _S]
    lib.bto_gemver_pass2_async.restype = c_int
    lib.bto_gemver_pass2_async.argtypes = [_P, _P, _D, _P, _L, _L, _S]
    for name in ("axpydot", "bicgk", "atax", "gemver"):
        sfn = getattr(lib, f"bto_{name}_sharded_async")
        sfn.restype = c_int
        sfn.argtypes = [_CT[ch] for ch in SIGNATURES[name]] + [_S]
    lib.bto_prim_matvec_async.restype = c_int
    lib.bto_prim_matvec_async.argtypes = [_P, _P, _P, _L, _L, c_int, _S]
    lib.bto_prim_axpby_async.restype = c_int
    lib.bto_prim_axpby_async.argtypes = [_D, _P, _D, _P, _P, _L, c_int, _S]
    lib.bto_prim_outer_async.restype = c_int
    lib.bto_prim_outer_async.argtypes = [_P, _P, _P, _L, _L, _S]
    lib.bto_prim_dot_async.restype = c_int
    lib.bto_prim_dot_async.argtypes = [_P, _P, _P, _L, _S]
    lib.bto_colsum_axpz_async.restype = c_int
    lib.bto_colsum_axpz_async.argtypes = [_P, _P, _D, _P, _P, _L, _L, _S]
    lib.bto_rank2_rowdot_async.restype = c_int
    lib.bto_rank2_rowdot_async.argtypes = [_P, _P, _P, _P, _P, _P, _D, _P, _P, _P, _L, _L, _S]
    lib.bto_exchange_init.restype = c_int
    lib.bto_exchange_init.argtypes = [c_int, c_int, POINTER(c_void_p), POINTER(c_void_p), _L,
                                      ctypes.c_uint]
    lib.bto_exchange_shutdown.restype = c_int
    lib.bto_exchange_flag_bytes.restype = c_int
    lib.bto_exchange_flag_bytes.argtypes = [c_int]
    lib.bto_exchange_status.restype = c_int
    lib.bto_exchange_status.argtypes = [POINTER(ctypes.c_uint)]
    lib.bto_last_launch_signature.restype = ctypes.c_ulonglong
    lib.bto_last_launch_plan.restype = c_char_p
    lib.bto_reserve_workspace.restype = c_int
    lib.bto_reserve_workspace.argtypes = [_S, _L]
    lib.bto_last_error.restype = c_int
    lib.bto_last_error_string.restype = c_char_p
    lib.bto_clear_error.restype = None
    lib.bto_abi_version.restype = c_int
    lib.bto_set_stream.restype = c_int
    lib.bto_set_stream.argtypes = [_S]
    lib.bto_set_tuning.restype = c_int
    lib.bto_set_tuning.argtypes = [c_char_p, _L]
    lib.bto_get_tuning.restype = _L
    lib.bto_get_tuning.argtypes = [c_char_p]
    lib.bto_kernel_launches.restype = _L
    lib.bto_bytes_min.restype = _D
    lib.bto_bytes_min.argtypes = [c_char_p, _L, _L]
    lib.bto_device_info.restype = c_int
    lib.bto_device_info.argtypes = [POINTER(c_int), POINTER(c_int),
                                    POINTER(_L), POINTER(_L)]
    lib.bto_workspace_bytes.restype = _L
    lib.bto_release_workspace.restype = c_int
    lib.bto_copy_to_device.restype = c_int
    lib.bto_copy_to_device.argtypes = [_P, _P, _L]
    lib.bto_copy_to_host.restype = c_int
    lib.bto_copy_to_host.argtypes = [_P, _P, _L]
    lib.bto_debug_poison_shared_memory.restype = c_int
    lib.bto_debug_poison_shared_memory.argtypes = [_S]
    lib.bto_debug_poison_all.restype = c_int
    lib.bto_debug_poison_all.argtypes = []
    lib.bto_debug_poison_workspace.restype = c_int
    lib.bto_debug_poison_workspace.argtypes = [_S]
    lib.bto_fill_host.restype = c_int
    lib.bto_fill_host.argtypes = [_P, _L, _D]
    _lib = lib
    return lib


def check(rc: int | None = None) -> None:
    """Raise BtoError on a non-zero return code, or -- for the void section-1
    symbols -- on a non-zero bto_last_error()."""
    lib = load()
    code = lib.bto_last_error() if rc is None else rc
    if code != 0:
        raise BtoError(code, lib.bto_last_error_string().decode(errors="replace"))


def set_tuning(**kv: int) -> None:
    lib = load()
    for key, value in kv.items():
        check(lib.bto_set_tuning(key.encode(), int(value)))


def get_tuning(key: str) -> int:
    return int(load().bto_get_tuning(key.encode()))


def kernel_launches() -> int:
    return int(load().bto_kernel_launches())


def launch_signature() -> int:
    """Hash of the kernel instances the last library call of this thread launched."""
    return int(load().bto_last_launch_signature())


def poison_shared_memory() -> None:
    """Testing hook: every SM's shared memory := NaN bit patterns, on torch's current stream."""
    import torch
    check(load().bto_debug_poison_shared_memory(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))


def poison_all() -> None:
    """Testing hook: shared memory on the library's stream and every stream's workspace := NaN patterns
    (what the host-pointer entry points run on)."""
    check(load().bto_debug_poison_all())


def poison_workspace() -> None:
    """Testing hook: the current stream's partial-sum workspace := NaN bit patterns."""
    import torch
    check(load().bto_debug_poison_workspace(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))


def launch_plan() -> str:
    """Kernel instances (names with template arguments) the last library call launched."""
    return load().bto_last_launch_plan().decode()


def bytes_min(kernel: str, M: int, N: int = 1) -> float:
    value = float(load().bto_bytes_min(kernel.lower().encode(), int(M), int(N)))
    if value < 0:
        raise KeyError(f"unknown kernel {kernel!r}")
    return value


def device_info() -> dict:
    lib = load()
    sm, thr = c_int(0), c_int(0)
    l2, mem = _L(0), _L(0)
    check(lib.bto_device_info(ctypes.byref(sm), ctypes.byref(thr),
                              ctypes.byref(l2), ctypes.byref(mem)))
    return {"sm_count": sm.value, "max_threads_per_sm": thr.value,
            "l2_bytes": l2.value, "global_bytes": mem.value}


def to_device(array):
    """numpy float64 array -> new CUDA tensor through the library's staged copy (pageable
    memory at 45-50 GB/s; torch's own pageable copy runs at ~11 GB/s on this platform)."""
    import ctypes

    import numpy as np
    import torch
    a = np.ascontiguousarray(array, dtype=np.float64)
    t = torch.empty(a.shape, dtype=torch.float64, device="cuda")
    torch.cuda.current_stream().synchronize()
    check(load().bto_copy_to_device(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(a.ctypes.data), a.nbytes))
    return t


def to_host(tensor):
    """Contiguous float64 CUDA tensor -> new numpy array through the staged copy."""
    import ctypes

    import numpy as np
    import torch
    t = tensor.contiguous()
    out = np.empty(tuple(t.shape), dtype=np.float64)
    torch.cuda.current_stream().synchronize()
    check(load().bto_copy_to_host(ctypes.c_void_p(out.ctypes.data), ctypes.c_void_p(t.data_ptr()), out.nbytes))
    return out


def filled(size: int, value: float):
    """np.full(size, value) with the first touch of the pages done by the copy threads."""
    import ctypes

    import numpy as np
    out = np.empty(int(size), dtype=np.float64)
    check(load().bto_fill_host(ctypes.c_void_p(out.ctypes.data), out.size, float(value)))
    return out
