#!/usr/bin/env python
"""Time the per-rank work of the row-sharded suite for G = 1, 2, 4, 8 on ONE GPU (the shard of
rank 0: rows M/G x N), i.e. everything of a strong-scaling step except the exchange."""
import json, statistics, sys
from pathlib import Path
import torch
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import bench
from paper_1205_1098_b200 import sharded, _native

class NoComm:
    def all_reduce_sum(self, t): pass
sharded.TorchComm = NoComm
torch.cuda.set_device(0)
_native.load()
rows = []
for G in (1, 2, 4, 8):
    suite = bench.Suite(torch, 0, G, bench.SUITE)
    for name in bench.SUITE:
        for _ in range(5):
            suite.launch(name)
        torch.cuda.synchronize()
        evs = []
        for _ in range(25):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); suite.launch(name); b.record(); evs.append((a, b))
        torch.cuda.synchronize()
        us = statistics.median(a.elapsed_time(b) for a, b in evs) * 1e3
        nbytes = bench.bytes_min(name, *bench.BENCH[name]) / G
        rows.append({"G": G, "kernel": name, "us": us, "gbs_per_gpu": nbytes / us / 1e3})
        print(f"G={G} {name:8s} shard {us:9.1f} us  {nbytes / us / 1e3:7.0f} GB/s per GPU", flush=True)
    del suite
    torch.cuda.empty_cache()
(REPO / "gpurun_out").mkdir(exist_ok=True)
(REPO / "gpurun_out" / "shard_scan.json").write_text(json.dumps(rows, indent=1))
