#!/usr/bin/env python
"""Snapshot loop IRs of the reference for a spread of organisms (build container only).

For each corpus kernel: the max-fuse organism, the unfused one, and seeded random
legal organisms (the reference's own `random_organism`, as in its acceptance
criterion 1, tests/test_acceptance.py:66-76), lowered + contracted by the reference
(`contract_arrays(lower(org, g))`) and stored as plain dicts through
`paper_1205_1098_b200.cuemit.ir_from_matfuse`.  The GPU tests emit CUDA from these
snapshots, so organism-driven emission is exercised on machines without the reference.

Run:  python tests/golden/make_organisms.py      -> tests/golden/organisms.json
"""
from __future__ import annotations

import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent.parent))

from matfuse import contract_arrays, lower, max_fuse  # noqa: E402
from matfuse.corpus import load_graph  # noqa: E402
from matfuse.fuse import canonical_key, fusion_legal, initial_forest  # noqa: E402
from matfuse.search import SearchConfig, random_organism  # noqa: E402

from paper_1205_1098_b200 import CORPUS  # noqa: E402
from paper_1205_1098_b200.cuemit import ir_from_matfuse  # noqa: E402

RANDOM_PER_KERNEL = 10


def main():
    cfg = SearchConfig(core_count=8)
    out = {}
    for name in CORPUS:
        g = load_graph(name)
        rng = random.Random(1234)
        organisms = {}
        for org in (max_fuse(g, 8), initial_forest(g)):
            organisms.setdefault(canonical_key(org), org)
        draws = 0
        while len(organisms) < 2 + RANDOM_PER_KERNEL and draws < 400:
            org = random_organism(g, rng, cfg, steps=rng.randrange(1, 14))
            draws += 1
            if fusion_legal(org, g) is None:
                organisms.setdefault(canonical_key(org), org)
        out[name] = [ir_from_matfuse(contract_arrays(lower(org, g))) for org in organisms.values()]
        print(f"{name}: {len(out[name])} organisms")
    path = HERE / "organisms.json"
    path.write_text(json.dumps(out, separators=(",", ":")))
    print(f"{path}: {path.stat().st_size / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
