#!/usr/bin/env python
"""Per-launch times of kernel sequences (no medians) to see carry-over effects."""
import sys
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from bench import Suite  # noqa: E402
from paper_1205_1098_b200 import _native  # noqa: E402

torch.cuda.set_device(0)
_native.load()
suite = Suite(torch, 0, 1, ("axpydot", "bicgk", "atax", "gesummv", "gemver"))
for _ in range(3):
    for k in ("axpydot", "bicgk", "atax", "gesummv", "gemver"):
        suite.launch(k)
torch.cuda.synchronize()


def run(seq):
    evs = []
    for k in seq:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if k == "sleep":
            torch.cuda._sleep(4_000_000)
        else:
            suite.launch(k)
        b.record()
        evs.append((k, a, b))
    torch.cuda.synchronize()
    print("  ".join(f"{k[:4]}:{a.elapsed_time(b):.3f}" for k, a, b in evs), flush=True)


for seq in (["atax"] * 10, ["gesummv"] + ["atax"] * 5, ["gemver"] + ["atax"] * 5,
            ["bicgk"] + ["atax"] * 5, ["sleep"] + ["atax"] * 5,
            ["gesummv", "atax"] * 4, ["bicgk", "atax"] * 4, ["gesummv", "bicgk", "atax"] * 3,
            ["axpydot"] * 8, ["sleep"] + ["axpydot"] * 5, ["bicgk", "axpydot"] * 4,
            ["axpydot", "bicgk", "atax", "gesummv", "gemver"] * 3):
    run(seq)
