#!/usr/bin/env python
"""Time the per-rank work of the row-sharded suite for G = 1, 2, 4, 8 on ONE GPU (the shard of
rank 0: rows M/G x N), i.e. everything of a strong-scaling step except the exchange: per
sequence issued eagerly and replayed from its captured CUDA graph (what bench.py --gpus N does),
and the whole step of five graphs back to back."""
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
    suite = bench.Suite(torch, 0, G, bench.SUITE, exchange="nccl")
    graphs = {}
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
        replay = suite.runner.capture(lambda name=name: suite._launch_eager(name))
        graphs[name] = replay
        evs = []
        for _ in range(25):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); replay(); b.record(); evs.append((a, b))
        torch.cuda.synchronize()
        us_graph = statistics.median(a.elapsed_time(b) for a, b in evs) * 1e3
        nbytes = bench.bytes_min(name, *bench.BENCH[name]) / G
        rows.append({"G": G, "kernel": name, "us": us, "us_graph": us_graph, "gbs_per_gpu": nbytes / us / 1e3,
                     "gbs_per_gpu_graph": nbytes / us_graph / 1e3})
        print(f"G={G} {name:8s} shard eager {us:9.1f} us {nbytes / us / 1e3:7.0f} GB/s | graph {us_graph:9.1f} us "
              f"{nbytes / us_graph / 1e3:7.0f} GB/s per GPU", flush=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        for name in bench.SUITE:
            graphs[name]()
    torch.cuda.synchronize()
    a.record()
    for _ in range(20):
        for name in bench.SUITE:
            graphs[name]()
    b.record()
    torch.cuda.synchronize()
    step_us = a.elapsed_time(b) * 1e3 / 20
    total = sum(bench.bytes_min(k, *bench.BENCH[k]) for k in bench.SUITE) / G
    rows.append({"G": G, "kernel": "step", "us_graph": step_us, "gbs_per_gpu_graph": total / step_us / 1e3})
    print(f"G={G} step (5 graphs back to back) {step_us:9.1f} us  {total / step_us / 1e3:7.0f} GB/s per GPU", flush=True)
    del graphs
    del suite
    torch.cuda.empty_cache()
(REPO / "gpurun_out").mkdir(exist_ok=True)
(REPO / "gpurun_out" / "shard_scan.json").write_text(json.dumps(rows, indent=1))
