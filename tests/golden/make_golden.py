#!/usr/bin/env python
"""Generate tests/golden/*.npz from the REFERENCE itself (build container only).

Imports matfuse from /root/reference/pkg/src (read-only; it cannot travel to
the GPU box, hence these committed fixtures) and records, per corpus kernel:

  small/<M>x<N>/s<seed>/O1/<out>   reference_evaluate           (interp.py:100)
  small/<M>x<N>/s<seed>/O2/<out>   generated C, max_fuse(g, 8)  (runtime.py:99)
      for the reference's own criterion-1 extent pairs
      (tests/test_acceptance.py:60-63) + two ragged ones, inputs from the
      reference's random_inputs (runtime.py:153) at seeds 0..2;
  check/O1|O2/<out>                the BASELINE.json check config (hot path
      only), inputs = SURVEY 8d generator (scalars U[-1,1)), seeds 0..4.
      Vector outputs are stored whole; outputs above 16 Ki elements are stored
      as a sha256 of their bytes plus a 4096-element strided sample.
  */inputs_sha                     sha256 over the generated inputs, so a
      drifting generator is caught before a parity test blames a kernel.

Run:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

from matfuse import contract_arrays, emit_c, lower, max_fuse, reference_evaluate  # noqa: E402
from matfuse.corpus import load_graph  # noqa: E402
from matfuse.runtime import Toolchain, random_inputs, run_kernel, workdir  # noqa: E402

import paper_1205_1098_b200 as bto  # noqa: E402

SMALL = [(1, 1), (1, 7), (7, 1), (2, 2), (7, 50), (50, 200), (200, 200),
         (13, 9), (33, 515)]
SMALL_SEEDS = (0, 1, 2)
BIG = 1 << 14


def sha(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).tobytes())
    return h.hexdigest()


def inputs_sha(graph, inputs) -> str:
    return sha([inputs[n] for n, _ in graph.spec.inputs])


def put(store: dict, prefix: str, outputs: dict):
    for name, value in outputs.items():
        arr = np.asarray(value, dtype=np.float64)
        if arr.size > BIG:
            flat = arr.ravel()
            step = flat.size // 4096
            store[f"{prefix}/{name}__sha"] = np.array(sha([arr]))
            store[f"{prefix}/{name}__sample"] = flat[::step][:4096].copy()
            store[f"{prefix}/{name}__step"] = np.array(step)
        else:
            store[f"{prefix}/{name}"] = arr


def main():
    tc = Toolchain()
    for name in bto.CORPUS:
        g = load_graph(name)
        mine = bto.load_graph(name)
        ker = emit_c(contract_arrays(lower(max_fuse(g, 8), g)))
        so = tc.compile(ker.source, workdir(), shared=True)
        store: dict = {"organism": np.array(ker.organism_key)}
        vector_only = g.extent_names == ("M",)
        pairs = sorted({(m, 1) for m, _ in SMALL} | {(n, 1) for _, n in SMALL}) \
            if vector_only else SMALL
        for (m, n) in pairs:
            ext = {"M": m} if vector_only else {"M": m, "N": n}
            for seed in SMALL_SEEDS:
                inp = random_inputs(g, ext, seed=seed)
                # our generator must reproduce the reference's bit for bit
                ours = bto.random_inputs(mine, ext, seed=seed)
                assert inputs_sha(g, inp) == inputs_sha(g, ours), (name, ext)
                key = f"small/{m}x{n}/s{seed}"
                store[f"{key}/inputs_sha"] = np.array(inputs_sha(g, inp))
                put(store, f"{key}/O1", reference_evaluate(g.spec, inp))
                put(store, f"{key}/O2", run_kernel(so, ker, g, inp, ext))
        if name in bto.CHECK_CONFIGS:
            ext = bto.CHECK_CONFIGS[name]
            inp = bto.gen_inputs(mine, ext, seed=bto.SEEDS[name])
            store["check/inputs_sha"] = np.array(inputs_sha(g, inp))
            put(store, "check/O1", reference_evaluate(g.spec, inp))
            put(store, "check/O2", run_kernel(so, ker, g, inp, ext))
        np.savez_compressed(HERE / f"{name}.npz", **store)
        print(f"{name}: {len(store)} arrays, "
              f"{(HERE / (name + '.npz')).stat().st_size / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
