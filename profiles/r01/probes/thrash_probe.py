#!/usr/bin/env python
"""Why is a kernel slower inside the suite than when it is re-run alone?  Time one
kernel preceded (untimed) by different kinds of traffic."""
import statistics
import sys
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from bench import BENCH, Suite, bytes_min  # noqa: E402
from paper_1205_1098_b200 import _native  # noqa: E402

torch.cuda.set_device(0)
_native.load()
suite = Suite(torch, 0, 1, ("axpydot", "bicgk", "atax", "gesummv", "gemver"))
other = torch.empty(3 * (1 << 30), dtype=torch.float64, device="cuda")      # 24 GiB elsewhere
page_idx = torch.arange(0, other.numel(), (2 << 20) // 8, device="cuda")    # one element per 2 MiB page


def touch_pages():
    other[page_idx] += 1.0          # ~12k scattered accesses: TLB traffic, no bandwidth


def big_read():
    other[: 1 << 30].sum()          # 8 GiB read of other memory


def big_write():
    other[: 1 << 30].zero_()        # 8 GiB write


PRE = {"none": lambda: None, "touch_pages": touch_pages, "big_read": big_read, "big_write": big_write,
       "bicgk": lambda: suite.launch("bicgk"), "gesummv": lambda: suite.launch("gesummv"),
       "gemver": lambda: suite.launch("gemver"), "atax": lambda: suite.launch("atax"),
       "sleep": lambda: torch.cuda._sleep(4_000_000)}

for name in ("axpydot", "atax", "bicgk"):
    for pre_name, pre in PRE.items():
        for _ in range(3):
            pre()
            suite.launch(name)
        evs = []
        for _ in range(11):
            pre()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            suite.launch(name)
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in evs)
        print(f"{name:8s} after {pre_name:12s}: {ms:.4f} ms  "
              f"{bytes_min(name, *BENCH[name]) / ms / 1e6:7.1f} GB/s", flush=True)
