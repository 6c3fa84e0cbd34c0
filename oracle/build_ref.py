#!/usr/bin/env python
"""Compile the REFERENCE's own CPU implementation of the hot path into oracle/_ref/.

TEST INFRASTRUCTURE (see oracle/bto_oracle.c).  The reference (matfuse) has no
kernel sources on disk: its emitter prints C99+OpenMP for an organism at run
time with the thread count baked into the pragma (cemit.py:190-193).  This
script imports the reference from /root/reference/pkg/src (read-only, never
copied), asks it for `max_fuse(graph, t)` (search.py:195) -> `lower` ->
`contract_arrays` -> `emit_c` for every corpus kernel and a ladder of thread
counts, and compiles each with the reference's own Toolchain template
(`cc -O3 -fopenmp ... -shared -fPIC -DMATFUSE_NO_MAIN`, runtime.py:26,70-83).

Outputs (generated C, .so, manifest.json) go ONLY into oracle/_ref/, which is
git-ignored but travels to the GPU box with the snapshot.  On the GPU box
/root/reference does not exist: tests and bench.py only dlopen the prebuilt
.so files listed in manifest.json.
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_SRC = Path(os.environ.get("BTO_REFERENCE_SRC", "/root/reference/pkg/src"))
OUT = HERE / "_ref"

KERNELS = ("axpydot", "bicgk", "atax", "gesummv", "gemver",
           "vadd", "waxpby", "dgemv", "dgemvt", "batax")
# thread ladder: the bench picks the largest entry <= os.cpu_count()
THREADS = (1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 112, 128, 160, 192,
           224, 256)


def main() -> int:
    if not REF_SRC.exists():
        print(f"build_ref: {REF_SRC} not present; nothing to do", file=sys.stderr)
        return 0
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF_SRC))
    from matfuse import contract_arrays, emit_c, lower, max_fuse
    from matfuse.corpus import load_graph
    from matfuse.fuse import initial_forest
    from matfuse.runtime import Toolchain

    OUT.mkdir(exist_ok=True)
    tc = Toolchain()
    manifest = {"template": tc.template, "cc": tc.cc, "kernels": {}}
    for name in KERNELS:
        graph = load_graph(name)
        entry = {
            "params": None,
            "inputs": [[n, d.kind] for n, d in graph.spec.inputs],
            "outputs": [[n, d.kind] for n, d in graph.spec.outputs],
            "dims": {n: list(graph.data[n].dims)
                     for n, _ in graph.spec.inputs + graph.spec.outputs},
            "extent_names": list(graph.extent_names),
            "variants": {},
        }
        jobs = [(f"t{t}", max_fuse(graph, t)) for t in THREADS]
        jobs.append(("unfused", initial_forest(graph)))
        for tag, org in jobs:
            ker = emit_c(contract_arrays(lower(org, graph)))
            stem = f"{name}_{tag}"
            so = tc.compile(ker.source, OUT, name=stem, shared=True)
            entry["params"] = [logical for _, logical in ker.params]
            entry["variants"][tag] = {
                "so": so.name, "organism": ker.organism_key,
                "threads": list(ker.threads), "symbol": ker.kernel_name,
            }
        manifest["kernels"][name] = entry
        print(f"build_ref: {name}: {len(jobs)} variants")
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
