"""ctypes access to the CPU oracle (oracle/) -- TEST INFRASTRUCTURE ONLY.

Two checkers live behind this module:
  * the hand restatement  oracle/libbto_oracle.so  (`oracle_run`), thread count
    chosen at run time;
  * the reference's own generated C  oracle/_ref/*.so  (`ref_run`), prebuilt in
    the build container by oracle/build_ref.py with the thread count baked in.
Nothing under paper_1205_1098_b200/ imports this.
"""
from __future__ import annotations

import ctypes
import json
import subprocess
from pathlib import Path

import numpy as np

ORACLE_DIR = Path(__file__).resolve().parent.parent / "oracle"
ORACLE_SO = ORACLE_DIR / "libbto_oracle.so"
REF_DIR = ORACLE_DIR / "_ref"

# C argument order of every kernel = the reference's kernel_params order
# (cemit.py:225-241).  'a' array in, 's' scalar in, 'o' array out, 'r' scalar out.
PARAMS = {
    "axpydot": [("w", "a"), ("v", "a"), ("u", "a"), ("alpha", "s"), ("z", "o"), ("beta", "r")],
    "bicgk": [("A", "a"), ("p", "a"), ("r", "a"), ("q", "o"), ("s", "o")],
    "atax": [("A", "a"), ("x", "a"), ("y", "o")],
    "gesummv": [("alpha", "s"), ("beta", "s"), ("A", "a"), ("B", "a"), ("x", "a"), ("y", "o")],
    "gemver": [("A", "a"), ("u1", "a"), ("v1", "a"), ("u2", "a"), ("v2", "a"),
               ("alpha", "s"), ("beta", "s"), ("y", "a"), ("z", "a"),
               ("B", "o"), ("x", "o"), ("w", "o")],
    "vadd": [("w", "a"), ("y", "a"), ("z", "a"), ("x", "o")],
    "waxpby": [("alpha", "s"), ("x", "a"), ("beta", "s"), ("y", "a"), ("w", "o")],
    "dgemv": [("alpha", "s"), ("A", "a"), ("x", "a"), ("beta", "s"), ("y", "a"), ("z", "o")],
    "dgemvt": [("alpha", "s"), ("beta", "s"), ("A", "a"), ("y", "a"), ("z", "a"),
               ("x", "o"), ("w", "o")],
    "batax": [("x", "a"), ("beta", "s"), ("A", "a"), ("y", "o")],
}
# output shapes in terms of extents
OUT_DIMS = {
    "axpydot": {"z": ("M",), "beta": ()},
    "bicgk": {"q": ("M",), "s": ("N",)},
    "atax": {"y": ("N",)},
    "gesummv": {"y": ("M",)},
    "gemver": {"B": ("M", "N"), "x": ("N",), "w": ("M",)},
    "vadd": {"x": ("M",)},
    "waxpby": {"w": ("M",)},
    "dgemv": {"z": ("M",)},
    "dgemvt": {"x": ("N",), "w": ("M",)},
    "batax": {"y": ("N",)},
}
VECTOR_ONLY = ("axpydot", "vadd", "waxpby")

_oracle = None
_ref_libs: dict = {}
_manifest = None


def ensure_built() -> Path:
    if not ORACLE_SO.exists() or \
            ORACLE_SO.stat().st_mtime < (ORACLE_DIR / "bto_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-C", str(ORACLE_DIR)], check=True,
                       capture_output=True)
    return ORACLE_SO


def _lib():
    global _oracle
    if _oracle is None:
        ensure_built()
        _oracle = ctypes.CDLL(str(ORACLE_SO))
    return _oracle


def max_threads() -> int:
    fn = _lib().bto_oracle_max_threads
    fn.restype = ctypes.c_int
    return int(fn())


def _bind(fn, name: str, inputs: dict, extents: dict, trailing: list, outputs: dict | None = None):
    """Marshal once; returns (thunk, collect): thunk() runs the C function on
    the prebuilt argument list (what the CPU baseline times), collect() reads
    the outputs back as the reference's run_kernel would return them.
    `outputs` may hand over preallocated flat float64 buffers by output name (the CPU
    baseline at bench size re-uses an 8 GiB buffer instead of allocating another)."""
    args, keep, outs = [], [], {}
    for pname, cls in PARAMS[name]:
        if cls == "s":
            args.append(ctypes.c_double(float(inputs[pname])))
        elif cls == "a":
            flat = np.ascontiguousarray(np.asarray(inputs[pname], dtype=np.float64).ravel())
            keep.append(flat)
            args.append(flat.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        else:
            size = 1
            for d in OUT_DIMS[name][pname]:
                size *= int(extents[d])
            buf = (outputs or {}).get(pname)
            if buf is None:
                buf = np.full(size, np.nan)
            assert buf.dtype == np.float64 and buf.size >= size and buf.flags.c_contiguous
            outs[pname] = buf
            args.append(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    names = ("M",) if name in VECTOR_ONLY else ("M", "N")
    args += [ctypes.c_long(int(extents[e])) for e in names] + trailing
    fn.restype = None

    def thunk():
        fn(*args)

    def collect():
        result = {}
        for pname, buf in outs.items():
            dims = OUT_DIMS[name][pname]
            shape = tuple(int(extents[d]) for d in dims)
            result[pname] = float(buf[0]) if not dims else \
                buf[:int(np.prod(shape))].reshape(shape)
        return result

    thunk.keep = keep
    return thunk, collect


def _call(fn, name: str, inputs: dict, extents: dict, trailing: list):
    thunk, collect = _bind(fn, name, inputs, extents, trailing)
    thunk()
    return collect()


def bind_oracle(name: str, inputs: dict, extents: dict, threads: int, outputs: dict | None = None):
    return _bind(getattr(_lib(), f"oracle_{name}"), name, inputs, extents,
                 [ctypes.c_int(int(threads))], outputs)


def bind_ref(name: str, inputs: dict, extents: dict, tag: str, outputs: dict | None = None):
    fn, _ = ref_function(name, tag)
    return _bind(fn, name, inputs, extents, [], outputs)


def oracle_run(name: str, inputs: dict, extents: dict, threads: int = 8) -> dict:
    """The hand restatement (oracle/bto_oracle.c) at `threads` blocks."""
    fn = getattr(_lib(), f"oracle_{name}")
    return _call(fn, name, inputs, extents, [ctypes.c_int(int(threads))])


def ref_manifest() -> dict | None:
    global _manifest
    if _manifest is None and (REF_DIR / "manifest.json").exists():
        _manifest = json.loads((REF_DIR / "manifest.json").read_text())
    return _manifest


def ref_available() -> bool:
    return ref_manifest() is not None


def ref_thread_ladder(name: str) -> list[int]:
    variants = ref_manifest()["kernels"][name]["variants"]
    return sorted(int(tag[1:]) for tag in variants if tag.startswith("t"))


def ref_run(name: str, inputs: dict, extents: dict, tag: str = "t8") -> dict:
    """The reference's generated C (prebuilt .so under oracle/_ref)."""
    info = ref_manifest()["kernels"][name]["variants"][tag]
    key = (name, tag)
    if key not in _ref_libs:
        _ref_libs[key] = ctypes.CDLL(str(REF_DIR / info["so"]))
    fn = getattr(_ref_libs[key], info["symbol"])
    return _call(fn, name, inputs, extents, [])


def ref_function(name: str, tag: str):
    """(ctypes function, info) for timing the reference .so directly."""
    info = ref_manifest()["kernels"][name]["variants"][tag]
    key = (name, tag)
    if key not in _ref_libs:
        _ref_libs[key] = ctypes.CDLL(str(REF_DIR / info["so"]))
    fn = getattr(_ref_libs[key], info["symbol"])
    fn.restype = None
    return fn, info
