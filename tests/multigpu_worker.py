"""One rank of the real multi-GPU parity run (launched by tests/test_multigpu.py under torch's
launcher, one process per GPU; TEST INFRASTRUCTURE -- the oracle is the checker here).

Every reduced sequence (AXPYDOT, BiCGK, ATAX, GEMVER) and the exchange-free GESUMMV run on
this rank's row shard through `ShardedRunner`, once with the NCCL all-reduce and once with the
exchange fused into the join kernel over NVLink peer memory, eagerly and as replayed CUDA
graphs; the gathered results are compared with the unsharded CPU oracle on rank 0 and must
be bit-identical across ranks.  Prints one JSON line per rank 0."""
from __future__ import annotations

import json
import math
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))

import oracle_lib  # noqa: E402
import paper_1205_1098_b200 as bto  # noqa: E402
from paper_1205_1098_b200.sharded import (SHARDING, GpuShardOps, NvlinkExchange, ShardedRunner,  # noqa: E402
                                          TorchComm, fused_exchange_agrees, row_block, shard_inputs)

SHAPES = [(1031, 2050), (4096, 4096), (777, 33000)]


def main() -> int:
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ops, comm = GpuShardOps(), TorchComm()
    report = {"world": world, "cases": 0, "fused": None, "worst": 0.0}
    modes = [("nccl", ShardedRunner(ops, comm, rank, world, fused=False))]
    exchange = None
    try:
        exchange = NvlinkExchange(max_vector=max(max(s) for s in SHAPES))
        assert fused_exchange_agrees(ops, comm, rank, world), "fused exchange disagrees with NCCL on the probe"
        modes.append(("fused", ShardedRunner(ops, comm, rank, world, fused=True)))
        report["fused"] = "ok"
    except Exception as exc:                         # no symmetric memory on this box: NCCL only, said so
        report["fused"] = f"unavailable: {type(exc).__name__}: {exc}"

    def dev(v):
        return torch.from_numpy(np.ascontiguousarray(v)).cuda() if isinstance(v, np.ndarray) else v

    for (m, n) in SHAPES:
        for name in ("axpydot", "bicgk", "atax", "gesummv", "gemver"):
            graph = bto.load_graph(name)
            ext = {"M": m * 37} if name == "axpydot" else {"M": m, "N": n}
            rows = ext["M"]
            full = bto.gen_inputs(graph, ext, seed=bto.SEEDS[name])          # same on every rank
            want = oracle_lib.oracle_run(name, full, ext, threads=8) if rank == 0 else None
            mine = {k: dev(v) for k, v in shard_inputs(name, full, rank, world, rows).items()}
            lo, hi = row_block(rows, rank, world)
            nan = lambda *shape: torch.full(shape, float("nan"), dtype=torch.float64, device="cuda")
            for label, runner in modes:
                for graphed in (False, True):
                    if name == "axpydot":
                        outs = {"z": nan(hi - lo), "beta": nan(1)}
                        call = lambda: runner.axpydot(mine["w"], mine["v"], mine["u"], mine["alpha"], outs["z"], outs["beta"])
                    elif name == "bicgk":
                        outs = {"q": nan(hi - lo), "s": nan(n)}
                        call = lambda: runner.bicgk(mine["A"], mine["p"], mine["r"], outs["q"], outs["s"])
                    elif name == "atax":
                        outs = {"y": nan(n)}
                        call = lambda: runner.atax(mine["A"], mine["x"], outs["y"])
                    elif name == "gesummv":
                        outs = {"y": nan(hi - lo)}
                        call = lambda: runner.gesummv(mine["alpha"], mine["beta"], mine["A"], mine["B"], mine["x"], outs["y"])
                    else:
                        outs = {"B": nan(hi - lo, n), "x": nan(n), "w": nan(hi - lo)}
                        colsum = nan(n)
                        call = lambda: runner.gemver(mine["A"], mine["u1"], mine["v1"], mine["u2"], mine["v2"],
                                                     mine["alpha"], mine["beta"], mine["y"], mine["z"],
                                                     outs["B"], outs["x"], outs["w"], colsum)
                    if graphed:
                        replay = runner.capture(call)
                        for t in outs.values():
                            t.fill_(float("nan"))
                        replay()
                        replay()                     # consecutive epochs / both buffer halves
                    else:
                        call()
                    torch.cuda.synchronize()
                    spec = SHARDING[name]
                    got = {}
                    for out_name, t in outs.items():
                        if out_name in spec.sharded_out:
                            sizes = [row_block(rows, r, world) for r in range(world)]
                            parts = [torch.empty((b - a,) + tuple(t.shape[1:]), dtype=torch.float64, device="cuda")
                                     for a, b in sizes]
                            dist.all_gather(parts, t.contiguous())
                            got[out_name] = torch.cat(parts).cpu().numpy()
                        else:
                            copies = [torch.empty_like(t) for _ in range(world)]
                            dist.all_gather(copies, t)
                            for c in copies[1:]:
                                assert torch.equal(c, copies[0]), f"{name}.{out_name} ({label}): ranks disagree"
                            got[out_name] = t.cpu().numpy() if t.numel() > 1 else float(t[0])
                    if rank == 0:
                        err = bto.max_rel_error(got, want)
                        tol = 1e-12 * max(1.0, math.log2(max(ext.values())))
                        assert err <= tol, f"{name} {ext} {label} graphed={graphed}: {err:.3e} > {tol:.3e}"
                        for o in {"axpydot": ("z",), "gemver": ("B",)}.get(name, ()):
                            assert np.array_equal(got[o], want[o]), f"{name}.{o} not bit-exact ({label})"
                        report["worst"] = max(report["worst"], err)
                        report["cases"] += 1
    if exchange is not None and report["fused"] == "ok":
        report["exchanges"] = exchange.status()
        exchange.close()
    dist.barrier()
    if rank == 0:
        print(json.dumps(report))
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
