#!/usr/bin/env python
"""bench.py -- BASELINE.json's metric on a B200: effective HBM GB/s of the fused kernels.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--kernel suite|axpydot|bicgk|atax|gesummv|gemver] [--no-e2e]
                    [--exchange auto|nccl|fused]

A "step" is one pass of the hot path over the suite: the five fused sequences
at BASELINE.json's bench sizes (AXPYDOT n=2^27; BiCGK, ATAX, GEMVER n=32768;
GESUMMV n=24576), fp64, seeded synthetic inputs generated on the device.
`value` = (sum of the sequences' minimum-traffic bytes) / (device
time of the step), inputs resident in HBM; every input is >= 4 GiB >> L2
(126 MB), so no L2 flush is needed between iterations.

Extra objects on the JSON line: `per_kernel` (achieved GB/s of each sequence),
`roofline` (the slowest-by-share sequence against MEASURED_PEAKS.json),
`e2e` (the same suite through the reference-facing C symbols with PINNED HOST
buffers, copies inside the timed region), `cpu_baseline` (the reference's own
generated C on this box's cores at the SAME sizes, plus the unfused organism on
a smaller sample), `clocks`, `gpu_launches`.

N > 1: `python bench.py --gpus N` starts N ranks itself (torchrun's launcher,
127.0.0.1) when it is not already running under one; it fails loudly when fewer
than N GPUs are visible.  Rows are sharded over ranks
(paper_1205_1098_b200.sharded), one exchange per kernel -- fused into the join
kernel over NVLink peer memory when symmetric memory is available and agrees
with NCCL on a probe, else one NCCL all-reduce -- and each rank's step is a
replayed CUDA graph.  Total problem size fixed -> "scaling": "strong".

`--impl reference` times the reference's CPU implementation (oracle/_ref, the
generated C compiled in the build container; else the oracle port) on the
host cores, same metric, same sizes; rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import re
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

SUITE = ("axpydot", "bicgk", "atax", "gesummv", "gemver")
BENCH = {"axpydot": (1 << 27, 1), "bicgk": (32768, 32768), "atax": (32768, 32768),
         "gesummv": (24576, 24576), "gemver": (32768, 32768)}
# fallback when the host cannot hold the bench sizes (needs ~17 GiB): out of last-level cache
CPU_SAMPLE = {"axpydot": (1 << 26, 1), "bicgk": (16384, 16384), "atax": (16384, 16384),
              "gesummv": (12288, 12288), "gemver": (16384, 16384)}
# the unfused organism (fuse.py:128 initial_forest) is serial and allocates a matrix per statement
UNFUSED_SAMPLE = {"axpydot": (1 << 25, 1), "bicgk": (8192, 8192), "atax": (8192, 8192),
                  "gesummv": (6144, 6144), "gemver": (8192, 8192)}

METRIC = "effective HBM GB/s (min bytes/time), fused suite"
WORKLOAD = ("suite5: AXPYDOT n=2^27, BiCGK n=32768, ATAX n=32768, GESUMMV n=24576, "
            "GEMVER n=32768")


def describe(sizes: dict, kernels) -> str:
    if sizes is BENCH or all(sizes[k] == BENCH[k] for k in kernels):
        return WORKLOAD if tuple(kernels) == SUITE else \
            "; ".join(f"{k} at BASELINE bench size {list(BENCH[k])}" for k in kernels)
    return "REDUCED sizes (not the BASELINE bench sizes): " + \
        ", ".join(f"{k} {sizes[k][0]}" + ("" if k == "axpydot" else f"x{sizes[k][1]}") for k in kernels)


def config_of(kernels, world: int, sizes=BENCH) -> dict:
    """The `config` object -- identical for the b200 and the reference arm of one run."""
    return {
        "workload": describe(sizes, kernels),
        "parallelism": "unsharded (1 rank)" if world == 1 else f"row-shard x{world} (strong scaling)",
        "l2": "every input >= 4 GiB >> 126 MB L2 (and any host LLC); no flush between iterations",
    }


def bytes_min(kernel: str, M: int, N: int) -> float:
    """SURVEY.md section 8d (same table as bto_bytes_min in the library)."""
    m, n = float(M), float(N)
    return {"axpydot": 32 * m, "bicgk": 8 * m * n + 16 * m + 16 * n,
            "atax": 8 * m * n + 16 * n, "gesummv": 16 * m * n + 8 * n + 8 * m,
            "gemver": 24 * m * n + 32 * m + 40 * n}[kernel]


def measured_peak() -> tuple[float, str]:
    path = REPO / "MEASURED_PEAKS.json"
    if path.exists():
        try:
            return float(json.loads(path.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks during the timed region

class ClockSampler:
    BAD = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown"}
    NOTE = {0x4: "sw_power_cap", 0x80: "hw_power_brake", 0x1: "gpu_idle",
            0x2: "app_clocks", 0x100: "display", 0x10: "sync_boost"}

    def __init__(self, index: int = 0, period: float = 0.05):
        self.index, self.period = index, period
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _loop(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in {**self.BAD, **self.NOTE}.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._thread = threading.Thread(target=self._loop, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": int(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons)}


# ---------------------------------------------------------------------------
# CPU arm: the reference's generated C (oracle/_ref) or the oracle port

def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def fill_uniform(arr, seed: int, threads: int) -> None:
    """arr[:] = U[-1,1) with `threads` independent PCG64 streams (numpy releases the GIL)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    flat = arr.reshape(-1)
    piece = 1 << 22
    jobs = [(lo, min(lo + piece, flat.size)) for lo in range(0, flat.size, piece)]

    def work(job):
        lo, hi = job
        view = flat[lo:hi]
        np.random.Generator(np.random.PCG64([seed, lo])).random(out=view)
        np.multiply(view, 2.0, out=view)
        np.subtract(view, 1.0, out=view)

    with ThreadPoolExecutor(max(1, threads)) as pool:
        list(pool.map(work, jobs))


class HostWorkset:
    """Host operands of the suite at `sizes`: two matrix-sized buffers that every sequence
    borrows views of (what e2e_host and the CPU arm both run on), plus the vectors."""

    def __init__(self, sizes, kernels, alloc=None, filled: bool = True):
        import numpy as np
        self.np = np
        self.sizes = sizes
        mats = [sizes[k][0] * sizes[k][1] for k in kernels if k != "axpydot"]
        need = max(mats + [3 * sizes["axpydot"][0] if "axpydot" in kernels else 0])
        alloc = alloc or (lambda count: np.empty(count, dtype=np.float64))
        self.big_in, self.big_out = alloc(need), alloc(need)
        nmax = max(max(sizes[k]) for k in kernels if k != "axpydot") if mats else 1
        self.vec = [alloc(nmax) for _ in range(8)]
        self.outv = [alloc(nmax) for _ in range(3)]
        self.scalar = alloc(1)
        if filled:
            t = host_cores()
            fill_uniform(self.big_in, 11, t)
            fill_uniform(self.big_out, 12, t)
            for i, v in enumerate(self.vec):
                fill_uniform(v, 20 + i, 1)

    def operands(self, name: str):
        """(inputs by parameter name, preallocated outputs by name, extents) on views."""
        M, N = self.sizes[name]
        bi, bo, v, o = self.big_in, self.big_out, self.vec, self.outv
        if name == "axpydot":
            return ({"w": bi[:M], "v": bi[M:2 * M], "u": bi[2 * M:3 * M], "alpha": 0.37},
                    {"z": bo[:M], "beta": self.scalar}, {"M": M})
        A = bi[:M * N].reshape(M, N)
        ext = {"M": M, "N": N}
        if name == "bicgk":
            return {"A": A, "p": v[0][:N], "r": v[1][:M]}, {"q": o[0][:M], "s": o[1][:N]}, ext
        if name == "atax":
            return {"A": A, "x": v[0][:N]}, {"y": o[0][:N]}, ext
        if name == "gesummv":
            return ({"alpha": 0.61, "beta": -0.27, "A": A, "B": bo[:M * N].reshape(M, N), "x": v[0][:N]},
                    {"y": o[0][:M]}, ext)
        return ({"A": A, "u1": v[1][:M], "v1": v[2][:N], "u2": v[3][:M], "v2": v[4][:N],
                 "alpha": 0.83, "beta": -0.41, "y": v[5][:M], "z": v[6][:N]},
                {"B": bo[:M * N], "x": o[1][:N], "w": o[2][:M]}, ext)


def _time_cpu(O, tag_or_threads, use_ref: bool, work: HostWorkset, kernels, steps: int, warmup: int):
    per, tot_bytes, tot_sec = {}, 0.0, 0.0
    for name in kernels:
        inputs, outputs, ext = work.operands(name)
        run, _ = O.bind_ref(name, inputs, ext, tag_or_threads, outputs) if use_ref else \
            O.bind_oracle(name, inputs, ext, tag_or_threads, outputs)
        for _ in range(warmup):
            run()
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            run()
            times.append(time.perf_counter() - t0)
        sec = statistics.mean(times)
        M, N = work.sizes[name]
        b = bytes_min(name, M, N)
        per[name] = {"gbs": b / sec / 1e9, "ms": sec * 1e3, "ms_min": min(times) * 1e3, "extents": [M, N]}
        tot_bytes += b
        tot_sec += sec
    return per, tot_bytes, tot_sec


def host_memory_free_bytes() -> int:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def cpu_baseline(steps: int = 2, warmup: int = 1, kernels=SUITE, work: HostWorkset | None = None,
                 unfused: bool = True) -> dict:
    """The reference's CPU path on this box's cores: max_fuse(graph, cores) as generated C
    (cemit.py, OpenMP) at the BENCH sizes -- the same configuration the GPU arm runs -- and,
    as a second figure, the unfused organism (fuse.py:128 `initial_forest`, serial, one
    matrix-sized temporary per statement) next to the fused one on a smaller sample."""
    sys.path.insert(0, str(REPO / "tests"))
    import oracle_lib as O

    cores_avail = host_cores()
    use_ref = O.ref_available()
    if use_ref:
        ladder = O.ref_thread_ladder("bicgk")
        threads = max(t for t in ladder if t <= max(1, cores_avail))
        kind, how = "reference", f"t{threads}"
    else:
        O.ensure_built()
        threads = max(1, cores_avail)
        kind, how = "port", threads
    sizes = BENCH
    if work is None:
        need = 2 * 8 * max(BENCH[k][0] * BENCH[k][1] for k in kernels) + (1 << 30)
        if host_memory_free_bytes() and host_memory_free_bytes() < need:
            sizes = CPU_SAMPLE          # said so in config.workload: not the same configuration
        work = HostWorkset(sizes, kernels)
    else:
        sizes = work.sizes
    per, tot_bytes, tot_sec = _time_cpu(O, how, use_ref, work, kernels, steps, warmup)
    out = {"value": tot_bytes / tot_sec / 1e9, "unit": "GB/s", "cores": threads,
           "kind": kind, "ms_per_step": tot_sec * 1e3, "per_kernel": per, "sizes": sizes,
           "sample": "%s; the C function alone on preallocated host buffers (no copies, no allocation "
                     "of operands); mean of %d reps after %d warm-up, %d OpenMP threads"
                     % (describe(sizes, kernels), steps, warmup, threads)}
    if unfused and use_ref:
        try:
            small = HostWorkset(UNFUSED_SAMPLE, kernels)
            # the unfused organism writes its outputs AND its temporaries itself
            u_per, u_b, u_s = _time_cpu(O, "unfused", True, small, kernels, 1, 1)
            f1_per, f1_b, f1_s = _time_cpu(O, "t1", True, small, kernels, 1, 1)
            ft_per, ft_b, ft_s = _time_cpu(O, how, True, small, kernels, 1, 1)
            out["unfused"] = {
                "value": u_b / u_s / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference",
                "organism": "initial_forest(graph) (fuse.py:128): one loop nest per statement, serial",
                "per_kernel": {k: round(v["gbs"], 2) for k, v in u_per.items()},
                "fused_1_thread": {"value": f1_b / f1_s / 1e9,
                                   "per_kernel": {k: round(v["gbs"], 2) for k, v in f1_per.items()}},
                "fused_all_threads": {"value": ft_b / ft_s / 1e9, "cores": threads,
                                      "per_kernel": {k: round(v["gbs"], 2) for k, v in ft_per.items()}},
                "fusion_speedup_1_thread": (f1_b / f1_s) / (u_b / u_s),
                "sample": describe(UNFUSED_SAMPLE, kernels) + "; GB/s of the FUSED minimum bytes; 1 rep after 1 warm-up",
            }
            del small
        except Exception as exc:          # the fused figure stands on its own
            out["unfused"] = {"value": None, "error": f"{type(exc).__name__}: {exc}"}
    return out


def run_reference_arm(args) -> int:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    kernels = SUITE if args.kernel == "suite" else (args.kernel,)
    steps, warmup = max(1, args.steps), max(0, args.warmup)
    base = cpu_baseline(steps=steps, warmup=warmup, kernels=kernels)
    line = {
        "impl": "reference", "metric": METRIC,
        "value": base["value"], "unit": "GB/s", "n_gpus": args.gpus, "steps": steps,
        "warmup": warmup, "ms_per_step": base["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(kernels, max(1, args.gpus), base["sizes"]),
        "timing": "perf_counter around each C call, mean over the steps; rank 0's host cores only",
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "per_kernel": base["per_kernel"],
        "e2e": {"value": base["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    if "unfused" in base:
        line["cpu_baseline"]["unfused"] = base["unfused"]
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# GPU arm

class Suite:
    """Device buffers + launch closures for the five sequences on one rank."""

    def __init__(self, torch, rank: int, world: int, kernels, exchange: str = "auto"):
        from paper_1205_1098_b200 import _native
        from paper_1205_1098_b200.sharded import GpuShardOps, ShardedRunner, TorchComm, row_block
        self.torch, self.rank, self.world = torch, rank, world
        self.native = _native
        self.ops = GpuShardOps()
        comm = TorchComm() if world > 1 else None
        self.exchange_kind = "none" if world == 1 else "nccl all-reduce after the join"
        self.exchange = None
        fused = False
        if world > 1 and exchange in ("auto", "fused"):
            # join-fused NVLink exchange (include/bto_b200.h 3b) when symmetric memory is there AND
            # a probe agrees with NCCL bit for bit on every rank; otherwise the library all-reduce
            try:
                from paper_1205_1098_b200.sharded import NvlinkExchange, fused_exchange_agrees
                self.exchange = NvlinkExchange(max_vector=32768)
                if fused_exchange_agrees(self.ops, comm, rank, world):
                    fused, self.exchange_kind = True, "fused into the join kernel (NVLink peer memory)"
                else:
                    self.exchange_kind = "nccl all-reduce (fused exchange failed its probe)"
            except Exception as exc:
                self.exchange_kind = f"nccl all-reduce (fused exchange unavailable: {type(exc).__name__}: {exc})"
            if not fused and exchange == "fused":
                raise RuntimeError(f"--exchange fused requested but {self.exchange_kind}")
            if rank == 0 and not fused:
                print(f"[bench] {self.exchange_kind}", file=sys.stderr)
        self.runner = ShardedRunner(self.ops, comm, rank, world, fused=fused)
        self.replays = {}
        self.kernels = kernels
        dev = torch.device("cuda", torch.cuda.current_device())
        gen = torch.Generator(device=dev).manual_seed(1234 + rank)

        def rnd(*shape):
            return torch.rand(*shape, dtype=torch.float64, device=dev, generator=gen) * 2 - 1

        n = 32768
        lo, hi = row_block(n, rank, world)
        self.rows = hi - lo
        self.n = n
        need_mat = any(k in kernels for k in ("bicgk", "atax", "gemver", "gesummv"))
        if need_mat:
            self.A = rnd(self.rows, n)
            self.Bm = rnd(self.rows, n)            # GEMVER output; GESUMMV's 2nd input lives here
        # column-indexed vectors are REPLICATED: the same values on every rank
        rep = torch.Generator(device=dev).manual_seed(99)
        self.vecN = [torch.rand(n, dtype=torch.float64, device=dev, generator=rep) * 2 - 1
                     for _ in range(4)]            # p/x, v1, v2, z
        self.vecM = [rnd(self.rows) for _ in range(4)]   # r/y, u1, u2
        self.q = torch.empty(self.rows, dtype=torch.float64, device=dev)
        self.s = torch.empty(n, dtype=torch.float64, device=dev)
        self.x = torch.empty(n, dtype=torch.float64, device=dev)
        self.colsum = torch.empty(n, dtype=torch.float64, device=dev)
        self.w = torch.empty(self.rows, dtype=torch.float64, device=dev)
        # GESUMMV n = 24576 : views into the big buffers
        g = 24576
        glo, ghi = row_block(g, rank, world)
        self.grows, self.g = ghi - glo, g
        if "gesummv" in kernels:
            self.GA = self.A.view(-1)[: self.grows * g].view(self.grows, g)
            self.GB = self.Bm.view(-1)[: self.grows * g].view(self.grows, g)
            self.gy = torch.empty(self.grows, dtype=torch.float64, device=dev)
        # AXPYDOT n = 2^27 sliced over ranks
        a = 1 << 27
        alo, ahi = row_block(a, rank, world)
        self.an = ahi - alo
        if "axpydot" in kernels:
            self.aw, self.av, self.au = rnd(self.an), rnd(self.an), rnd(self.an)
            self.az = torch.empty(self.an, dtype=torch.float64, device=dev)
            self.abeta = torch.empty(1, dtype=torch.float64, device=dev)

    def operands(self, name: str):
        """(inputs, outputs) of this rank's shard of sequence `name`, as device tensors."""
        if name == "axpydot":
            return [self.aw, self.av, self.au], [self.az, self.abeta]
        if name == "bicgk":
            return [self.A, self.vecN[0], self.vecM[0]], [self.q, self.s]
        if name == "atax":
            return [self.A, self.vecN[0]], [self.s]
        if name == "gesummv":
            return [self.GA, self.GB, self.vecN[0][: self.g]], [self.gy]
        return ([self.A, self.vecM[1], self.vecN[1], self.vecM[2], self.vecN[2], self.vecM[0], self.vecN[3]],
                [self.Bm, self.x, self.w])

    def capture(self, name: str):
        """This rank's sequence `name`, exchange included, as a replayable CUDA graph."""
        self.replays[name] = self.runner.capture(lambda: self._launch_eager(name))
        return self.replays[name]

    def launch(self, name: str):
        replay = self.replays.get(name)
        if replay is not None:
            return replay()
        return self._launch_eager(name)

    def _launch_eager(self, name: str):
        r = self.runner
        if name == "axpydot":
            r.axpydot(self.aw, self.av, self.au, 0.37, self.az, self.abeta)
        elif name == "bicgk":
            r.bicgk(self.A, self.vecN[0], self.vecM[0], self.q, self.s)
        elif name == "atax":
            r.atax(self.A, self.vecN[0], self.s)
        elif name == "gesummv":
            r.gesummv(0.61, -0.27, self.GA, self.GB, self.vecN[0][: self.g], self.gy)
        elif name == "gemver":
            if self.world > 1:
                r.gemver(self.A, self.vecM[1], self.vecN[1], self.vecM[2], self.vecN[2], 0.83,
                         -0.41, self.vecM[0], self.vecN[3], self.Bm, self.x, self.w, self.colsum)
            else:
                self.ops.gemver(self.A, self.vecM[1], self.vecN[1], self.vecM[2], self.vecN[2],
                                0.83, -0.41, self.vecM[0], self.vecN[3], self.Bm, self.x, self.w)


def pinned_workset(torch, kernels) -> tuple[HostWorkset, str]:
    """Host operands in PINNED memory (pageable if the box's locked-memory limit says no),
    filled through the GPU's RNG (host RNG is slow); shared by e2e_host and the CPU leg."""
    kind = ["pinned"]
    keep = []

    def alloc(count):
        t = None
        if kind[0] == "pinned":
            try:
                t = torch.empty(count, dtype=torch.float64, pin_memory=True)
            except RuntimeError:          # locked-memory limit of the box: pageable host buffers
                kind[0] = "pageable (pinned allocation failed)"
        if t is None:
            t = torch.empty(count, dtype=torch.float64)
        keep.append(t)
        return t.numpy()

    work = HostWorkset(BENCH, kernels, alloc=alloc, filled=False)
    work.tensors = keep
    chunk = 1 << 26
    for t in keep:
        for off in range(0, t.numel(), chunk):
            n = min(chunk, t.numel() - off)
            t[off:off + n].copy_(torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1)
    torch.cuda.synchronize()
    return work, kind[0]


def e2e_host(torch, kernels, steps: int, warmup: int, work: HostWorkset, host_kind: str) -> dict:
    """The suite through the reference's C symbols with pinned HOST buffers:
    host->device copies of every input and device->host copies of every output
    are inside the timed region (the call returns when outputs are on the host)."""
    from paper_1205_1098_b200 import _native
    lib = _native.load()
    P = lambda a: ctypes.c_void_p(a.ctypes.data)
    order = {"axpydot": ("w", "v", "u", "alpha", "z", "beta"), "bicgk": ("A", "p", "r", "q", "s"),
             "atax": ("A", "x", "y"), "gesummv": ("alpha", "beta", "A", "B", "x", "y"),
             "gemver": ("A", "u1", "v1", "u2", "v2", "alpha", "beta", "y", "z", "B", "x", "w")}
    h2d = d2h = 0.0
    calls = []
    for k in kernels:
        ins, outs, ext = work.operands(k)
        args = []
        for name in order[k]:
            val = ins.get(name, outs.get(name))
            args.append(float(val) if isinstance(val, float) else P(val))
        args += [ext["M"]] + ([ext["N"]] if "N" in ext else [])
        calls.append((getattr(lib, k), args))
        h2d += sum(8.0 * v.size for v in ins.values() if not isinstance(v, float))
        d2h += sum(8.0 * v.size for v in outs.values())

    def step():
        for fn, args in calls:
            fn(*args)
            _native.check()

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        step()                                   # every call returns with its outputs on the host
        times.append(time.perf_counter() - t0)
    sec = statistics.median(times)               # (host-side hiccups: one step in ten runs 10 % long)
    total = sum(bytes_min(k, *BENCH[k]) for k in kernels)
    return {"value": total / sec / 1e9, "unit": "GB/s", "ms_per_step": sec * 1e3,
            "step_ms": [round(t * 1e3, 2) for t in times], "timing": "median step, wall clock",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": f"C symbols of include/bto_b200.h section 1 with {host_kind} host pointers"}


def e2e_sharded(torch, dist, suite, kernels, steps: int, warmup: int) -> dict:
    """N > 1: every rank pushes ITS shard of each sequence's inputs from pinned host memory, runs
    the sharded sequence (exchange included) and pulls its outputs back, blocking per sequence
    like a host-pointer call; whole-job bytes over the slowest rank's wall time."""
    mirrors = {}

    def host(t):
        key = (t.data_ptr(), t.numel())
        if key not in mirrors:
            mirrors[key] = torch.empty(t.numel(), dtype=torch.float64, pin_memory=True)
            mirrors[key].copy_(t.reshape(-1))
        return mirrors[key]

    plan = []
    h2d = d2h = 0.0
    for k in kernels:
        ins, outs = suite.operands(k)
        plan.append((k, [(t, host(t)) for t in ins], [(t, host(t)) for t in outs]))
        h2d += sum(8.0 * t.numel() for t in ins)
        d2h += sum(8.0 * t.numel() for t in outs)

    def step():
        for k, ins, outs in plan:
            for t, h in ins:
                t.view(-1).copy_(h, non_blocking=True) if t.is_contiguous() else t.copy_(h.view(t.shape), non_blocking=True)
            suite.launch(k)
            for t, h in outs:
                h.copy_(t.reshape(-1), non_blocking=True)
            torch.cuda.synchronize()

    for _ in range(warmup):
        step()
    if suite.world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    sec = (time.perf_counter() - t0) / steps
    if suite.world > 1:
        t = torch.tensor([sec, h2d, d2h], dtype=torch.float64, device="cuda")
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        sec, h2d, d2h = t.tolist()
    total = sum(bytes_min(k, *BENCH[k]) for k in kernels)
    return {"value": total / sec / 1e9, "unit": "GB/s", "ms_per_step": sec * 1e3,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": f"ShardedRunner on {suite.world} ranks, every rank's shard from / to pinned host memory"}


def normalise_kernel_name(name: str) -> str:
    """'void mv_tile_kernel<5, 8, 2, 1, 2>' (ncu) -> 'mv_tile_kernel<5,8,2,1,2>' (bto_last_launch_plan)."""
    name = name.strip()
    if name.startswith("void "):
        name = name[5:]
    return name.replace(" ", "")


def traffic_for(sequence: str, plan: str):
    """DRAM bytes of `sequence` from the committed ncu capture (profiles/traffic.json) -- but only
    if that capture profiled the kernel instances the library launches NOW (`plan`); a capture
    of other instances is reported as stale, never quoted."""
    try:
        tj = json.loads((REPO / "profiles" / "traffic.json").read_text())
        entry = tj[sequence]
    except Exception as exc:
        return None, f"unavailable ({type(exc).__name__})"
    # (the cluster size of the single-pass ATAX follows how many clusters the box's GPCs hold --
    #  8 or 9 at the bench size; its DRAM traffic does not depend on it, the kernel body is the same)
    same_body = lambda name: re.sub(r"^(atax_cluster_kernel<)\d+,", r"\1C,", name)
    launched = {same_body(k) for k in plan.split("+")} if plan else set()
    captured = {same_body(normalise_kernel_name(k)) for k in entry["kernels"]}
    if not captured <= launched:
        return None, f"stale: profiles/traffic.json profiled {sorted(captured)}, the library launches {plan}"
    return entry["dram_bytes"], tj["_source"]


def run_gpu_arm(args) -> int:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                                   f"(python bench.py --gpus N starts them itself)"}))
        return 2
    if not torch.cuda.is_available() or torch.cuda.device_count() <= local_rank:
        print(json.dumps({"error": "no CUDA device for this rank; this bench has no CPU fallback",
                          "n_gpus_requested": args.gpus, "n_gpus_visible": torch.cuda.device_count()
                          if torch.cuda.is_available() else 0}))
        return 2
    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    kernels = SUITE if args.kernel == "suite" else (args.kernel,)

    from paper_1205_1098_b200 import _native
    _native.load()
    suite = Suite(torch, rank, world, kernels, exchange=args.exchange)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    plans = {}
    for k in kernels:                      # first eager call: which kernel instances does it launch?
        suite.launch(k)
        plans[k] = _native.launch_plan()
    launches_per_step = 0
    if world > 1 or os.environ.get("BTO_BENCH_GRAPH"):
        # a rank's step is 90-500 us of kernels at 8 GPUs: replay captured graphs (kernels +
        # exchange), do not issue 2-5 launches and a collective per sequence from Python
        before = _native.kernel_launches()
        for k in kernels:
            suite._launch_eager(k)
        launches_per_step = _native.kernel_launches() - before
        for k in kernels:
            suite.capture(k)
    barrier()

    for _ in range(max(3, args.warmup)):
        for k in kernels:
            suite.launch(k)
    barrier()

    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in kernels] for _ in range(args.steps)]
    first, last = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _native.kernel_launches()
    with ClockSampler(local_rank) as clocks:
        barrier()
        first.record()
        for s in range(args.steps):
            for i, k in enumerate(kernels):
                ev[s][i][0].record()
                suite.launch(k)
                ev[s][i][1].record()
        last.record()
        barrier()
    launches = _native.kernel_launches() - launches0
    if suite.replays:                      # graph replays launch the captured kernels: count those
        launches = launches_per_step * args.steps
    if suite.exchange is not None and suite.runner.fused:
        suite.exchange.status()            # raises if a peer wait ran into the guard
    total_ms = first.elapsed_time(last)
    per_ms = {k: statistics.mean(ev[s][i][0].elapsed_time(ev[s][i][1]) for s in range(args.steps))
              for i, k in enumerate(kernels)}
    per_min = {k: min(ev[s][i][0].elapsed_time(ev[s][i][1]) for s in range(args.steps))
               for i, k in enumerate(kernels)}
    if world > 1:
        t = torch.tensor([total_ms] + [per_ms[k] for k in kernels], dtype=torch.float64,
                         device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        vals = t.tolist()
        total_ms = vals[0]
        per_ms = dict(zip(kernels, vals[1:]))
    sharded_e2e = None
    if (world > 1 or os.environ.get("BTO_BENCH_SHARDED_E2E")) and not args.no_e2e:
        try:
            sharded_e2e = e2e_sharded(torch, dist, suite, kernels, steps=max(1, min(args.steps, 3)), warmup=1)
        except Exception as exc:  # e.g. not enough pinned host memory
            sharded_e2e = {"value": None, "error": f"{type(exc).__name__}: {exc}"}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    ms_per_step = total_ms / args.steps
    total_bytes = sum(bytes_min(k, *BENCH[k]) for k in kernels)
    value = total_bytes / (ms_per_step * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    per_kernel = {}
    for k in kernels:
        gbs = bytes_min(k, *BENCH[k]) / (per_ms[k] * 1e-3) / 1e9
        per_kernel[k] = {"gbs": round(gbs, 1), "ms": round(per_ms[k], 4),
                         "ms_min": round(per_min[k], 4),
                         "frac_of_peak": round(gbs / (peak * world), 4),
                         "bytes_min": bytes_min(k, *BENCH[k]), "extents": list(BENCH[k])}
    dominant = max(kernels, key=lambda k: per_ms[k])
    dom = per_kernel[dominant]
    for k in kernels:
        per_kernel[k]["kernels"] = plans[k]
    traffic, traffic_src = (traffic_for(dominant, plans[dominant]) if world == 1
                            else (None, "single-GPU capture only"))
    line = {
        "metric": METRIC,
        "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config_of(kernels, world),
        "timing": "CUDA events on the launch stream, max over ranks",
        "exchange": suite.exchange_kind,
        "issue": "CUDA graph replay per sequence" if suite.replays else "eager launches",
        "per_kernel": per_kernel,
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": dom["gbs"],
                     "peak": peak * world, "unit": "GB/s",
                     "frac": round(dom["gbs"] / (peak * world), 4),
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                     "algorithmic_bytes": dom["bytes_min"],
                     "nominal_peak": 8000.0 * world,         # BASELINE.json north_star: ~8 TB/s per GPU
                     "frac_nominal": round(dom["gbs"] / (8000.0 * world), 4),
                     "peak_note": "the measured peak is a read+write copy; read-dominated kernels "
                                  "reach 7.1-7.5 TB/s on this part, hence fractions above 1"},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
    }
    line["suite_frac_of_peak"] = round(value / (peak * world), 4)
    line["suite_frac_of_nominal_8tbs"] = round(value / (8000.0 * world), 4)
    if sharded_e2e is not None:
        line["e2e"] = sharded_e2e
    work = None
    if world == 1 and sharded_e2e is None and not args.no_e2e:
        try:
            del suite                                   # the device copies: e2e stages its own
            work, host_kind = pinned_workset(torch, kernels)
            line["e2e"] = e2e_host(torch, kernels, steps=max(1, min(args.steps, 3)), warmup=1,
                                   work=work, host_kind=host_kind)
        except Exception as exc:  # e.g. not enough pinned host memory
            line["e2e"] = {"value": None, "error": f"{type(exc).__name__}: {exc}"}
    if world == 1 and not args.no_cpu:
        try:
            base = cpu_baseline(steps=2, warmup=1, kernels=kernels, work=work)
            line["cpu_baseline"] = {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")}
            line["cpu_baseline"]["per_kernel"] = {k: round(v["gbs"], 2)
                                                  for k, v in base["per_kernel"].items()}
            if "unfused" in base:
                line["cpu_baseline"]["unfused"] = base["unfused"]
        except Exception as exc:
            line["cpu_baseline"] = {"value": None, "error": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sock:
        sock.bind(("127.0.0.1", 0))
        return sock.getsockname()[1]


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` outside a launcher: start N ranks (one per GPU) with torch's
    launcher on 127.0.0.1 and pass their output through.  Fewer than N visible GPUs is an
    error -- never a silent N = 1 run."""
    import torch
    visible = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if visible < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested, {visible} CUDA device(s) visible",
                          "n_gpus_requested": args.gpus, "n_gpus_visible": visible}))
        return 3
    env = dict(os.environ)
    # leave NCCL's communicator lines on (rank count), on stderr so that stdout stays one JSON line
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--kernel", choices=("suite",) + SUITE, default="suite")
    ap.add_argument("--exchange", choices=("auto", "nccl", "fused"), default="auto",
                    help="N > 1: the exchange fused into the join kernel over NVLink peer memory "
                         "(auto: when symmetric memory is available and a probe agrees with NCCL), "
                         "or one NCCL all-reduce after the join")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--tune", action="append", default=[], metavar="KEY=VALUE",
                    help="experiments only: a bto_set_tuning key (include/bto_b200.h section 4)")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    for kv in args.tune:
        from paper_1205_1098_b200 import _native
        key, value = kv.split("=")
        _native.set_tuning(**{key: int(value)})
    return run_gpu_arm(args)


if __name__ == "__main__":
    raise SystemExit(main())
