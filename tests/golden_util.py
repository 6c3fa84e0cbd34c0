"""Read tests/golden/*.npz (written by tests/golden/make_golden.py)."""
from __future__ import annotations

import hashlib
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def _npz(kernel: str):
    return np.load(GOLDEN / f"{kernel}.npz")


def small_cases(kernel: str) -> list[tuple[int, int, int]]:
    """(M, N, seed) of every stored small case."""
    out = set()
    for key in _npz(kernel).files:
        if key.startswith("small/") and key.endswith("/inputs_sha"):
            _, ext, seed, _ = key.split("/")
            m, n = ext.split("x")
            out.add((int(m), int(n), int(seed[1:])))
    return sorted(out)


def sha(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).tobytes())
    return h.hexdigest()


def inputs_sha(kernel: str, prefix: str) -> str:
    return str(_npz(kernel)[f"{prefix}/inputs_sha"])


def expected(kernel: str, prefix: str, which: str) -> dict:
    """Stored outputs under `<prefix>/<O1|O2>/`; large arrays come back as
    {"sha":..., "sample":..., "step":...} records."""
    data = _npz(kernel)
    root = f"{prefix}/{which}/"
    out: dict = {}
    for key in data.files:
        if not key.startswith(root):
            continue
        leaf = key[len(root):]
        if "__" in leaf:
            name, field = leaf.split("__")
            out.setdefault(name, {})[field] = data[key]
        else:
            out[leaf] = data[key]
    return out


def max_err(got: dict, want: dict) -> float:
    """matfuse's max_rel_error (runtime.py:167-175), on whole arrays where the
    fixture stores them and on the strided sample where it stores a digest."""
    worst = 0.0
    for name, exp in want.items():
        g = np.asarray(got[name], dtype=np.float64)
        if isinstance(exp, dict):
            step = int(exp["step"])
            g = g.ravel()[::step][:4096]
            e = np.asarray(exp["sample"], dtype=np.float64)
        else:
            e = np.asarray(exp, dtype=np.float64)
            g = g.reshape(e.shape)
        if e.size:
            worst = max(worst, float(np.max(np.abs(g - e) / np.maximum(np.abs(e), 1.0))))
    return worst


def bit_equal(got, exp) -> bool:
    """Bit equality against a stored array or digest record."""
    g = np.asarray(got, dtype=np.float64)
    if isinstance(exp, dict):
        return sha([g]) == str(exp["sha"])
    return np.array_equal(g.reshape(np.asarray(exp).shape), np.asarray(exp))
