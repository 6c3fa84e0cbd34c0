"""Build libbto_b200.so in-tree with nvcc for sm_100a (cross-compiles without a GPU).

    python -m paper_1205_1098_b200.build [--force] [--verbose]

The shared object lands next to this file (git-ignored, but it travels to the
GPU box with the repo snapshot).  One translation unit: csrc/api.cu includes
the kernel headers.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
OUT = PKG_DIR / "libbto_b200.so"
STAMP = PKG_DIR / ".libbto_b200.stamp"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found (set NVCC)")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + \
        [REPO / "include" / "bto_b200.h"]


def _digest() -> str:
    h = hashlib.sha256()
    h.update(" ".join(NVCC_FLAGS).encode())
    for path in _sources():
        h.update(path.name.encode())
        h.update(path.read_bytes())
    return h.hexdigest()


def build_library(force: bool = False, verbose: bool = False) -> Path:
    """Compile if sources changed since the last build; returns the .so path."""
    digest = _digest()
    if not force and OUT.exists() and STAMP.exists() and STAMP.read_text() == digest:
        return OUT
    cmd = [_nvcc(), *NVCC_FLAGS, "-I", str(REPO / "include"), "-I", str(CSRC),
           "-o", str(OUT), str(CSRC / "api.cu")]
    if verbose:
        cmd += ["-Xptxas", "-v"]
        print(" ".join(cmd), file=sys.stderr)
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if verbose:
        sys.stderr.write(proc.stderr)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{proc.stderr.strip()}")
    STAMP.write_text(digest)
    return OUT


if __name__ == "__main__":
    path = build_library(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(path)
