"""Row-sharded multi-GPU execution: one process per GPU, one all-reduce per kernel.

The reference parallelises by cutting ONE axis into static blocks
(`lo = ext*p/t, hi = ext*(p+1)/t`, cemit.py:195-196), giving each block its
own partial buffer for reductions that cross the cut and joining the
partials afterwards (lower.py:123-135, cemit.py:204-222).  This module lifts
that protocol one level: rank g of G owns rows [M*g/G, M*(g+1)/G) of every
matrix and of every row-indexed vector; column-indexed vectors are
replicated; the "join" is a sum all-reduce over NCCL/NVLink of the
column-indexed result:

    AXPYDOT  all vectors sliced           all-reduce 1 fp64   (beta)
    BiCGK    q stays sharded              all-reduce N fp64   (s)
    ATAX     --                           all-reduce N fp64   (y)
    GESUMMV  y stays sharded              none
    GEMVER   B, w stay sharded            all-reduce N fp64   (B'y) BETWEEN the passes

`local` is the per-shard compute: in production `GpuShardOps` (the C ABI on
this rank's device); the CPU tests inject a numpy implementation to exercise
the slicing / exchange logic over gloo.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

__all__ = ["row_block", "ShardSpec", "SHARDING", "ShardedRunner", "GpuShardOps",
           "NvlinkExchange", "TorchComm", "shard_inputs", "fused_exchange_agrees"]


def row_block(extent: int, rank: int, world: int) -> tuple[int, int]:
    """Rows owned by `rank`: the reference's block bounds (cemit.py:195-196)."""
    return (extent * rank) // world, (extent * (rank + 1)) // world


@dataclass(frozen=True)
class ShardSpec:
    row_sliced: tuple[str, ...]      # inputs/outputs indexed by the row axis (sliced)
    replicated: tuple[str, ...]      # column-indexed inputs (every rank holds all)
    reduced: tuple[str, ...]         # outputs that need the sum all-reduce
    sharded_out: tuple[str, ...]     # outputs that stay row-sharded


SHARDING = {
    "axpydot": ShardSpec(("w", "v", "u", "z"), (), ("beta",), ("z",)),
    "bicgk": ShardSpec(("A", "r", "q"), ("p",), ("s",), ("q",)),
    "atax": ShardSpec(("A",), ("x",), ("y",), ()),
    "gesummv": ShardSpec(("A", "B", "y"), ("x",), (), ("y",)),
    "gemver": ShardSpec(("A", "u1", "u2", "y", "B", "w"), ("v1", "v2", "z"),
                        ("x",), ("B", "w")),
}


def shard_inputs(name: str, inputs: dict, rank: int, world: int, rows: int) -> dict:
    """Slice full-size inputs down to what `rank` owns (used by tests/bench)."""
    lo, hi = row_block(rows, rank, world)
    spec = SHARDING[name]
    return {k: (v[lo:hi] if k in spec.row_sliced else v) for k, v in inputs.items()}


class ShardedRunner:
    """Runs one kernel on this rank's shard and performs the exchange.

    comm: an object with `all_reduce_sum(tensor_or_array)` (in place);
    local: shard compute with methods named after the kernels (see GpuShardOps);
    fused: when True (and world > 1) the exchange is done INSIDE the join kernel
    over NVLink peer memory (`local.<kernel>_sharded`, set up by NvlinkExchange)
    instead of a separate all-reduce.
    """

    def __init__(self, local, comm, rank: int, world: int, fused: bool = False):
        self.local, self.comm, self.rank, self.world = local, comm, rank, world
        self.fused = fused and world > 1

    def capture(self, method, *args, warmup: int = 2):
        """Capture one sharded sequence (`method`: the name of one of this runner's methods, or any
        callable that issues library calls on the current stream) -- its kernels AND its exchange
        (the NCCL all-reduce or the join-fused NVLink exchange) -- into a CUDA graph and return
        `replay()`.

        At 8 GPUs a shard's kernels take 90-500 us; issuing 2-5 launches plus a collective
        eagerly from Python costs a comparable amount of host time, a graph launch ~10 us.
        The library's entry points are capture-safe (per-stream workspace that never moves
        under a captured kernel, exchange epoch on the device: include/bto_b200.h section 2);
        `warmup` eager calls run first on a side stream so that workspaces, occupancy caches
        and the communicator are set up outside the capture.  Every rank must capture and
        replay the same sequence the same number of times.  The operands must stay alive and
        in place for as long as the graph is replayed."""
        import torch
        fn = method if callable(method) else getattr(self, method)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                fn(*args)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            fn(*args)
        keep = (graph, args, side)

        def replay(_keep=keep):
            _keep[0].replay()
        replay.graph = graph
        return replay

    def axpydot(self, w, v, u, alpha, z, beta):
        if self.fused:
            return self.local.axpydot_sharded(w, v, u, alpha, z, beta)
        self.local.axpydot(w, v, u, alpha, z, beta)
        if self.world > 1:
            self.comm.all_reduce_sum(beta)

    def bicgk(self, A, p, r, q, s):
        if self.fused:
            return self.local.bicgk_sharded(A, p, r, q, s)
        self.local.bicgk(A, p, r, q, s)
        if self.world > 1:
            self.comm.all_reduce_sum(s)

    def atax(self, A, x, y):
        # t = A_g x is complete on the rank (rows are whole), y_g = A_g' t
        if self.fused:
            return self.local.atax_sharded(A, x, y)
        self.local.atax(A, x, y)
        if self.world > 1:
            self.comm.all_reduce_sum(y)

    def gesummv(self, alpha, beta, A, B, x, y):
        self.local.gesummv(alpha, beta, A, B, x, y)

    def gemver(self, A, u1, v1, u2, v2, alpha, beta, y, z, B, x, w, colsum):
        """colsum: N-element scratch for the exchanged B'y partials."""
        if self.fused:
            return self.local.gemver_sharded(A, u1, v1, u2, v2, alpha, beta, y, z, B, x, w)
        self.local.gemver_pass1(A, u1, v1, u2, v2, y, B, colsum)
        if self.world > 1:
            self.comm.all_reduce_sum(colsum)
        self.local.gemver_xupdate(colsum, beta, z, x)
        self.local.gemver_pass2(B, x, alpha, w)


class TorchComm:
    """Sum all-reduce through torch.distributed (NCCL on GPUs, gloo in tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def all_reduce_sum(self, tensor):
        self.dist.all_reduce(tensor, op=self.dist.ReduceOp.SUM, group=self.group)


class NvlinkExchange:
    """Symmetric exchange buffers for the join-fused all-reduce (include/bto_b200.h 3b).

    Allocates one symmetric-memory block per rank (torch.distributed._symmetric_memory:
    every rank maps every peer's block over NVLink), lays out
    [capacity doubles of exchange | world*64 u32 flags], zeroes it, and hands the
    peer pointers to the library.  Needs one process per GPU on an NVLink/NVSwitch
    node; there is no way to exercise it in a single-GPU environment, where the
    kernel itself is tested by emulating all ranks on one device
    (tests/test_gpu_parity.py::test_join_fused_exchange_emulated_ranks).
    """

    def __init__(self, max_vector: int, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        from . import _native

        lib = _native.load()
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        capacity = 2 * int(max_vector)
        flag_bytes = int(lib.bto_exchange_flag_bytes(self.world))
        total = capacity + (flag_bytes + 7) // 8
        self.block = symm_mem.empty(total, dtype=torch.float64, device=torch.device(
            "cuda", torch.cuda.current_device()))
        self.block.zero_()
        self.handle = symm_mem.rendezvous(self.block, group or dist.group.WORLD)
        torch.cuda.synchronize()
        dist.barrier(group)
        ptrs = [int(p) for p in self.handle.buffer_ptrs]
        exch = (ctypes.c_void_p * self.world)(*ptrs)
        flags = (ctypes.c_void_p * self.world)(*[p + 8 * capacity for p in ptrs])
        _native.check(lib.bto_exchange_init(self.rank, self.world, exch, flags, capacity, 0))
        self._lib, self._native = lib, _native

    def status(self) -> int:
        """Synchronise the device and raise BtoError if an exchange ran into the peer-wait guard
        (its results were set to NaN); returns the number of exchanges completed on this rank."""
        done = ctypes.c_uint(0)
        self._native.check(self._lib.bto_exchange_status(ctypes.byref(done)))
        return int(done.value)

    def close(self):
        self._native.check(self._lib.bto_exchange_shutdown())


def fused_exchange_agrees(ops, comm, rank: int, world: int, rows: int = 640, cols: int = 4100,
                          rounds: int = 3) -> bool:
    """Probe run before the fused exchange is trusted with a benchmark or a job: a small sharded
    BiCGK and AXPYDOT through `*_sharded` (exchange inside the join kernel) against the same shard
    through the plain entry point + `comm.all_reduce_sum`, `rounds` times (both parity halves of
    the exchange buffer, consecutive epochs).  True only if EVERY rank saw agreement within
    1e-12 relative (the two sums differ in order only), bit-identical results across ranks'
    own repeats, and a clean `bto_exchange_status`.  Needs bto_exchange_init (NvlinkExchange)."""
    import torch
    from . import _native
    gen = torch.Generator(device="cuda").manual_seed(4321 + rank)
    rep = torch.Generator(device="cuda").manual_seed(77)
    rnd = lambda g, *shape: torch.rand(*shape, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    A, r, p = rnd(gen, rows, cols), rnd(gen, rows), rnd(rep, cols)
    w, v, u = rnd(gen, 50001), rnd(gen, 50001), rnd(gen, 50001)
    ok = True
    try:
        want_s, want_b = torch.empty(cols, dtype=torch.float64, device="cuda"), torch.empty(1, dtype=torch.float64, device="cuda")
        q, z = torch.empty(rows, dtype=torch.float64, device="cuda"), torch.empty(50001, dtype=torch.float64, device="cuda")
        ops.bicgk(A, p, r, q, want_s)
        comm.all_reduce_sum(want_s)
        ops.axpydot(w, v, u, 0.37, z, want_b)
        comm.all_reduce_sum(want_b)
        first = None
        for _ in range(rounds):
            got_s = torch.full((cols,), float("nan"), dtype=torch.float64, device="cuda")
            got_b = torch.full((1,), float("nan"), dtype=torch.float64, device="cuda")
            ops.bicgk_sharded(A, p, r, q, got_s)
            ops.axpydot_sharded(w, v, u, 0.37, z, got_b)
            torch.cuda.synchronize()
            scale = torch.clamp(want_s.abs(), min=1.0)
            ok = ok and bool(((got_s - want_s).abs() / scale).max() <= 1e-12)
            ok = ok and bool(((got_b - want_b).abs() / torch.clamp(want_b.abs(), min=1.0)).max() <= 1e-12)
            if first is None:
                first = (got_s.clone(), got_b.clone())
            else:
                ok = ok and torch.equal(first[0], got_s) and torch.equal(first[1], got_b)
        done = ctypes.c_uint(0)
        ok = ok and _native.load().bto_exchange_status(ctypes.byref(done)) == 0
    except Exception:
        ok = False
    flag = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64, device="cuda")
    comm.all_reduce_sum(flag)
    return bool(flag.item() == float(world))


class GpuShardOps:
    """Per-shard compute through the asynchronous C ABI on the current stream.

    All arguments are contiguous float64 CUDA tensors on this rank's device
    (scalars are Python floats; `beta` of AXPYDOT is a 1-element tensor).
    """

    def __init__(self, stream=None):
        from . import _native
        self._native = _native
        self.lib = _native.load()
        self._stream = stream
        self._recording = None
        self._raw_stream = None

    def _st(self):
        # the raw handle of the current stream without building a torch.cuda.Stream object
        # (1.5 us -> 0.2 us; an eager mid-size call is bound by exactly this kind of cost)
        if self._stream is not None:
            return self._stream.cuda_stream
        if self._raw_stream is None:
            import torch
            self._raw_stream = torch._C._cuda_getCurrentRawStream
            self._current_device = torch.cuda.current_device
        return self._raw_stream(self._current_device())

    @staticmethod
    def _p(t):
        # a plain int: ctypes converts it through the declared argtype (c_void_p), which is
        # cheaper than constructing a c_void_p object per argument
        return t.data_ptr()

    def _call(self, fn, *args):
        if self._recording is not None:          # bind(): keep the marshalled call instead of making it
            self._recording.append((fn, args))
            return
        rc = fn(*args)
        if rc:
            self._native.check(rc)

    def bind(self, method: str, *args):
        """Pre-marshal one call: `f = ops.bind("bicgk", A, p, r, q, s)`, then `f()` launches it
        on the stream that was current at bind time, as often as wanted, without the per-call
        tensor -> pointer conversions (eager issue of a 2-launch sequence: ~16 -> ~9 us).  The
        tensors must stay alive and in place; a captured CUDA graph removes the rest."""
        self._recording = []
        try:
            getattr(self, method)(*args)
            recorded = self._recording
        finally:
            self._recording = None
        keep = args                                # hold the operands
        check = self._native.check
        if len(recorded) == 1:
            fn, cargs = recorded[0]
            return lambda _k=keep: check(fn(*cargs))

        def replay(_k=keep):
            for fn, cargs in recorded:
                check(fn(*cargs))
        return replay

    def axpydot(self, w, v, u, alpha, z, beta):
        self._call(self.lib.bto_axpydot_async, self._p(w), self._p(v), self._p(u), float(alpha), self._p(z), self._p(beta),
            w.numel(), self._st())

    def bicgk(self, A, p, r, q, s):
        self._call(self.lib.bto_bicgk_async, self._p(A), self._p(p), self._p(r), self._p(q), self._p(s),
            A.shape[0], A.shape[1], self._st())

    def atax(self, A, x, y):
        self._call(self.lib.bto_atax_async, self._p(A), self._p(x), self._p(y), A.shape[0], A.shape[1], self._st())

    def gesummv(self, alpha, beta, A, B, x, y):
        self._call(self.lib.bto_gesummv_async, float(alpha), float(beta), self._p(A), self._p(B), self._p(x), self._p(y),
            A.shape[0], A.shape[1], self._st())

    def gemver(self, A, u1, v1, u2, v2, alpha, beta, y, z, B, x, w):
        self._call(self.lib.bto_gemver_async, self._p(A), self._p(u1), self._p(v1), self._p(u2), self._p(v2),
            float(alpha), float(beta), self._p(y), self._p(z), self._p(B), self._p(x),
            self._p(w), A.shape[0], A.shape[1], self._st())

    # -- exchange fused into the join (needs NvlinkExchange / bto_exchange_init) --
    def axpydot_sharded(self, w, v, u, alpha, z, beta):
        self._call(self.lib.bto_axpydot_sharded_async, self._p(w), self._p(v), self._p(u), float(alpha), self._p(z), self._p(beta),
            w.numel(), self._st())

    def bicgk_sharded(self, A, p, r, q, s):
        self._call(self.lib.bto_bicgk_sharded_async, self._p(A), self._p(p), self._p(r), self._p(q), self._p(s),
            A.shape[0], A.shape[1], self._st())

    def atax_sharded(self, A, x, y):
        self._call(self.lib.bto_atax_sharded_async, self._p(A), self._p(x), self._p(y), A.shape[0], A.shape[1], self._st())

    def gemver_sharded(self, A, u1, v1, u2, v2, alpha, beta, y, z, B, x, w):
        self._call(self.lib.bto_gemver_sharded_async, self._p(A), self._p(u1), self._p(v1), self._p(u2), self._p(v2),
            float(alpha), float(beta), self._p(y), self._p(z), self._p(B), self._p(x),
            self._p(w), A.shape[0], A.shape[1], self._st())

    def gemver_pass1(self, A, u1, v1, u2, v2, y, B, colsum):
        self._call(self.lib.bto_gemver_pass1_async, self._p(A), self._p(u1), self._p(v1), self._p(u2), self._p(v2), self._p(y),
            self._p(B), self._p(colsum), A.shape[0], A.shape[1], self._st())

    def gemver_xupdate(self, colsum, beta, z, x):
        self._call(self.lib.bto_gemver_xupdate_async, self._p(colsum), float(beta), self._p(z), self._p(x), x.numel(), self._st())

    def gemver_pass2(self, B, x, alpha, w):
        self._call(self.lib.bto_gemver_pass2_async, self._p(B), self._p(x), float(alpha), self._p(w), B.shape[0], B.shape[1],
            self._st())
