"""Row-sharded multi-GPU runtime: host logic over gloo, world_size 2 and 3, CPU only.

The per-shard compute is injected (the oracle running on the shard), so these
tests exercise exactly what the multi-GPU runtime adds: the reference's block
bounds, which operands are sliced / replicated, where the single all-reduce
sits (between GEMVER's passes), and that the sharded result equals the
unsharded oracle within the reduction-order tolerance."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1205_1098_b200 as bto
from paper_1205_1098_b200.sharded import (SHARDING, ShardedRunner, TorchComm, row_block,
                                          shard_inputs)


def test_row_blocks_tile_the_extent():
    # the reference's formula (cemit.py:195-196): contiguous, disjoint, covering
    for extent in (1, 7, 8, 1000, 32768):
        for world in (1, 2, 3, 8):
            blocks = [row_block(extent, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == extent
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
    assert row_block(32768, 3, 8) == (12288, 16384)


def test_sharding_table_covers_every_operand():
    for name, spec in SHARDING.items():
        graph = bto.load_graph(name)
        declared = {n for n, d in graph.spec.inputs + graph.spec.outputs if d.kind != "scalar"}
        covered = set(spec.row_sliced) | set(spec.replicated) | set(spec.reduced)
        assert declared <= covered, (name, declared - covered)
        for n in spec.row_sliced:      # sliced operands are indexed by the row axis M
            assert graph.dims[n][0] == "M", (name, n)
        for n in spec.replicated:
            assert graph.dims[n] == ("N",), (name, n)


class OracleShardOps:
    """Shard compute on torch CPU tensors through the CPU oracle (test double for
    sharded.GpuShardOps)."""

    def __init__(self):
        import oracle_lib
        self.o = oracle_lib

    def _run(self, name, inputs, outs):
        ext = {"M": next(v.shape[0] for k, v in inputs.items() if hasattr(v, "shape") and
                         k in SHARDING.get(name, SHARDING["gemver"]).row_sliced)}
        for v in inputs.values():
            if hasattr(v, "shape") and v.ndim == 2:
                ext["N"] = v.shape[1]
        got = self.o.oracle_run(name, {k: (v.numpy() if hasattr(v, "numpy") else v)
                                       for k, v in inputs.items()}, ext, threads=1)
        for k, t in outs.items():
            t.copy_(torch.from_numpy(np.atleast_1d(np.asarray(got[k], dtype=np.float64))).reshape(t.shape))

    def axpydot(self, w, v, u, alpha, z, beta):
        self._run("axpydot", {"w": w, "v": v, "u": u, "alpha": alpha}, {"z": z, "beta": beta})

    def bicgk(self, A, p, r, q, s):
        self._run("bicgk", {"A": A, "p": p, "r": r}, {"q": q, "s": s})

    def atax(self, A, x, y):
        self._run("atax", {"A": A, "x": x}, {"y": y})

    def gesummv(self, alpha, beta, A, B, x, y):
        self._run("gesummv", {"alpha": alpha, "beta": beta, "A": A, "B": B, "x": x}, {"y": y})

    def gemver_pass1(self, A, u1, v1, u2, v2, y, B, colsum):
        B.copy_((A + torch.outer(u1, v1)) + torch.outer(u2, v2))
        colsum.copy_(B.t() @ y)

    def gemver_xupdate(self, colsum, beta, z, x):
        x.copy_(colsum * beta + z)

    def gemver_pass2(self, B, x, alpha, w):
        w.copy_((B @ x) * alpha)


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        runner = ShardedRunner(OracleShardOps(), TorchComm(), rank, world)
        M, N = 37, 29
        out = {}
        for name in ("axpydot", "bicgk", "atax", "gesummv", "gemver"):
            graph = bto.load_graph(name)
            ext = {"M": M} if name == "axpydot" else {"M": M, "N": N}
            full = bto.gen_inputs(graph, ext, seed=bto.SEEDS[name])
            mine = shard_inputs(name, full, rank, world, M)
            t = {k: (torch.from_numpy(np.ascontiguousarray(v)) if hasattr(v, "shape") else v)
                 for k, v in mine.items()}
            lo, hi = row_block(M, rank, world)
            rows = hi - lo
            z = lambda n: torch.full((n,), float("nan"), dtype=torch.float64)
            if name == "axpydot":
                zz, beta = z(rows), z(1)
                runner.axpydot(t["w"], t["v"], t["u"], t["alpha"], zz, beta)
                out[name] = {"z": zz, "beta": beta}
            elif name == "bicgk":
                q, s = z(rows), z(N)
                runner.bicgk(t["A"], t["p"], t["r"], q, s)
                out[name] = {"q": q, "s": s}
            elif name == "atax":
                y = z(N)
                runner.atax(t["A"], t["x"], y)
                out[name] = {"y": y}
            elif name == "gesummv":
                y = z(rows)
                runner.gesummv(t["alpha"], t["beta"], t["A"], t["B"], t["x"], y)
                out[name] = {"y": y}
            else:
                B, x, w, colsum = torch.full((rows, N), float("nan"), dtype=torch.float64), z(N), z(rows), z(N)
                runner.gemver(t["A"], t["u1"], t["v1"], t["u2"], t["v2"], t["alpha"], t["beta"],
                              t["y"], t["z"], B, x, w, colsum)
                out[name] = {"B": B, "x": x, "w": w}
        results[rank] = {k: {n: v.numpy().copy() for n, v in d.items()} for k, d in out.items()}
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_results_match_unsharded_oracle(oracle, world):
    manager = mp.Manager()
    results = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    M, N = 37, 29
    for name in ("axpydot", "bicgk", "atax", "gesummv", "gemver"):
        graph = bto.load_graph(name)
        ext = {"M": M} if name == "axpydot" else {"M": M, "N": N}
        want = oracle.oracle_run(name, bto.gen_inputs(graph, ext, seed=bto.SEEDS[name]), ext, threads=1)
        spec = SHARDING[name]
        for out_name, expected in want.items():
            if out_name in spec.sharded_out:      # concatenate the row shards
                got = np.concatenate([results[r][name][out_name] for r in range(world)], axis=0)
            else:                                 # reduced outputs: identical on every rank
                got = results[0][name][out_name]
                for r in range(1, world):
                    assert np.array_equal(results[r][name][out_name], got), (name, out_name)
            got = np.asarray(got).reshape(np.asarray(expected).shape) if np.ndim(expected) else float(got[0])
            err = bto.max_rel_error({out_name: got}, {out_name: expected})
            assert err < 1e-12, (name, out_name, err)
        # element-wise outputs stay bit-identical under sharding
        if name == "gemver":
            B = np.concatenate([results[r][name]["B"] for r in range(world)], axis=0)
            assert np.array_equal(B, want["B"])
