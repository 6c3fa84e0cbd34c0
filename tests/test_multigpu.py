"""Real multi-GPU runs (needs >= 2 B200s on one node; skipped otherwise -- the host logic is
covered on CPU by tests/test_sharded.py over gloo and the fused exchange kernel by the
emulated-rank test in tests/test_gpu_parity.py)."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

REPO = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _gpus() -> int:
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _clean_env() -> dict:
    return {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_sequences_on_real_peers(world):
    """NCCL and the join-fused NVLink exchange, eager and graph-replayed, for all four reduced
    sequences against the unsharded oracle; results bit-identical across ranks."""
    if _gpus() < world:
        pytest.skip(f"{_gpus()} GPU(s) visible, {world} needed")
    proc = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
                           str(_port()), str(REPO / "tests" / "multigpu_worker.py")],
                          capture_output=True, text=True, timeout=1500, env=_clean_env())
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    report = json.loads(proc.stdout.strip().splitlines()[-1])
    assert report["world"] == world and report["cases"] >= 3 * 5 * 2
    assert report["fused"] == "ok", report["fused"]       # an NVSwitch box must take the fused path


@pytest.mark.parametrize("world", [2, 4, 8])
def test_bench_starts_its_own_ranks(world):
    """`python bench.py --gpus N` with no launcher around it: N ranks, one JSON line, n_gpus = N."""
    if _gpus() < world:
        pytest.skip(f"{_gpus()} GPU(s) visible, {world} needed")
    proc = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", str(world), "--steps", "3",
                           "--warmup", "3", "--no-e2e"], capture_output=True, text=True, timeout=1500,
                          env=_clean_env())
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    lines = [l for l in proc.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["scaling"] == "strong" and d["issue"].startswith("CUDA graph")
    assert d["value"] > 3000.0 * world                    # >= ~45 % of the aggregate roofline even untuned
