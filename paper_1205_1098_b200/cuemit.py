"""CUDA emission for lowered kernels: the GPU counterpart of `matfuse.cemit`.

`cemit.emit_c` (cemit.py:250-291) prints C99 + OpenMP for ANY legal organism;
this module prints CUDA C for the same loop IR, so organism-driven code
generation also has a GPU back end.  The
hand-written sequences in csrc/ remain the fast path for the corpus kernels at
their best organisms; emitted kernels are correct for every organism and
reasonably parallel, not tuned.

Input: a plain-dict snapshot of the reference's `LoopIR` (`ir_from_matfuse`
takes the real object where the reference is importable; the dict is JSON-able,
which is how tests carry organisms to machines without the reference).

Mapping (the reference's emission rules, cemit.py:112-222, re-targeted):

* a parallel region (`IRParallel`, `#pragma omp parallel for` over blocks) becomes
  ONE kernel launch: block p of the partition is CTA p, same slice bounds
  `lo = ext*p/t, hi = ext*(p+1)/t`; `t` is the organism's thread count scaled up
  to fill the GPU (`blocks`), which the block formula allows for any t;
* inside a CTA every loop runs on all threads with identical bounds, except the
  INNERMOST loop of each nest, which is strided across the CTA's threads (it is
  the contiguous axis in the nests the reference derives, graph.py:504-546);
* a reduction statement inside a strided loop whose target is not indexed by that
  loop (row dots `q[i] += ..`, contracted scalars `t0_s += ..`, per-block partials)
  accumulates in a per-thread register and is combined with a fixed-order CTA
  reduction after the loop; thread 0 updates memory targets;
* statements outside strided loops run uniformly: contracted scalars in every
  thread, memory writes by thread 0; `__syncthreads()` separates the phases;
* partial buffers `[t x extent]` and the ascending join are as in the reference
  (cemit.py:183-222), the join being a small kernel;
* top-level items outside any region (serial code on the CPU) run in a single CTA.

The emitted translation unit exports `extern "C" void <kernel>(...)` with the
reference's argument order (cemit.py:225-241) taking DEVICE pointers; the call is
stream-ordered on the default stream (the caller synchronises, `run_emitted` does).
"""
from __future__ import annotations

import ctypes
import os
import shlex
import shutil
import subprocess
from dataclasses import dataclass
from pathlib import Path

from .runtime import GeneratedKernel, ToolchainError

__all__ = ["ir_from_matfuse", "emit_cuda", "emitted_kernel_for", "emitted_entry", "ir_for_spec", "NvccToolchain", "run_emitted", "DEFAULT_BLOCKS",
           "EMIT_VARIANTS", "time_emitted", "measure_empirical_ir", "OrganismTimer", "EmitModel", "estimate_cost_ir",
           "AnalyticOrganismCost"]

DEFAULT_BLOCKS = 592          # 4 CTAs per SM on a 148-SM part
CTA_THREADS = 256
SERIAL_THREADS = 1024


# ---------------------------------------------------------------------------
# IR snapshot

def ir_from_matfuse(ir) -> dict:
    """Snapshot a reference `LoopIR` (lower.py:78-93) as a JSON-able dict."""
    graph = ir.graph
    spec = graph.spec

    def item(it) -> dict:
        kind = type(it).__name__
        if kind == "IRStmt":
            return {"t": "stmt", "role": it.role, "op": it.op_id, "target": it.target}
        if kind == "IRLoop":
            return {"t": "loop", "axis": it.axis, "extent": it.extent, "sliced": bool(it.sliced),
                    "body": [item(b) for b in it.body]}
        return {"t": "par", "axis": it.axis, "extent": it.extent, "slot": it.slot,
                "partials": list(it.partials), "body": [item(b) for b in it.body]}

    from matfuse.fuse import canonical_key          # only reachable next to the reference
    return {
        "name": spec.name,
        "inputs": [[n, d.kind] for n, d in spec.inputs],
        "outputs": [[n, d.kind] for n, d in spec.outputs],
        "extents": list(graph.extent_names),
        "threads": list(ir.organism.threads),
        "organism": canonical_key(ir.organism),
        "storage": {n: {"cls": s.cls, "extents": list(s.extents), "labels": list(s.labels),
                        "order": s.order, "base": s.base} for n, s in ir.storage.items()},
        "ops": {str(op.op_id): {"kind": op.kind, "operands": [r.name for r in op.operands],
                                "result": op.result,
                                "reduction": op.nest.reduction_axis is not None}
                for op in graph.ops},
        "roots": [item(it) for it in ir.roots],
    }


# ---------------------------------------------------------------------------
# emitter

class _Writer:
    def __init__(self):
        self.lines: list[str] = []
        self.depth = 0

    def put(self, text: str = ""):
        self.lines.append("    " * self.depth + text if text else "")

    def open(self, text: str):
        self.put(text + " {" if text else "{")
        self.depth += 1

    def close(self, suffix: str = ""):
        self.depth -= 1
        self.put("}" + suffix)


_PRELUDE = r"""#include <cuda_runtime.h>

namespace {
// Batched loads of read-only operands.  `asm volatile` keeps them in program order ahead of
// the arithmetic (left to itself the compiler sinks each load to its use and the thread has
// one or two requests in flight instead of a whole batch).  Streamed-once data bypasses L1.
__device__ __forceinline__ double ld_stream(const double *p)
{
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_keep(const double *p)
{
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// fixed-order CTA reduction, result broadcast to every thread
__device__ __forceinline__ double cta_allreduce(double v, double *scratch)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double total = scratch[0];
    for (int w = 1; w < nwarps; ++w) total += scratch[w];
    return total;
}

// warp-level only (strip mode: every warp writes its own partial of a row dot, no CTA barrier)
template <int R>
__device__ __forceinline__ void warp_reduce_n(double (&v)[R])
{
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v[r] += __shfl_xor_sync(0xffffffffu, v[r], off);
    }
}

// the same for R values at once (R rows of an unrolled-and-jammed loop): one pair of
// barriers instead of R, every value summed in exactly the order cta_allreduce uses
template <int R>
__device__ __forceinline__ void cta_allreduce_n(double (&v)[R], double *scratch)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v[r] += __shfl_xor_sync(0xffffffffu, v[r], off);
    }
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) scratch[warp * R + r] = v[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double total = scratch[r];
        for (int w = 1; w < nwarps; ++w) total += scratch[w * R + r];
        v[r] = total;
    }
}

// Cluster mode (a region whose CTAs split the strided axis between the C CTAs of a cluster): a sum
// that leaves the axis is completed across the cluster.  Warp sums go to shared memory as in
// cta_allreduce_n; thread c < C then adds them (the CTA's total, warps in ascending order) and PUSHES
// it into CTA c's exchange buffer through distributed shared memory; ONE cluster barrier; every
// thread adds the C totals it finds in its own shared memory in rank order -- the same bits in
// every CTA.  Two buffers alternate (`par`): a peer overwrites a buffer only after the barrier of
// the exchange in between, which this CTA reaches after it has read it.
template <int R, int C>
__device__ __forceinline__ void cluster_allreduce_n(double (&v)[R], double *scratch, double *gather, int &par)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v[r] += __shfl_xor_sync(0xffffffffu, v[r], off);
    }
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) scratch[warp * R + r] = v[r];
    }
    __syncthreads();
    if (threadIdx.x < C) {
        unsigned rank, dst;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(dst) : "r"((unsigned)__cvta_generic_to_shared(gather + rank * R)), "r"(threadIdx.x));
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double total = scratch[r];
            for (int w = 1; w < nwarps; ++w) total += scratch[w * R + r];
            asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dst + 8u * r), "d"(total) : "memory");
        }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double total = gather[r];
#pragma unroll
        for (int c = 1; c < C; ++c) total += gather[c * R + r];
        v[r] = total;
    }
    par ^= 1;
}
}  // namespace
"""

JAM = 4                       # rows of an outer loop processed together (unroll-and-jam)
# Launch-shape variants an empirical timer may try per organism (B200 sweep at n = 8192,
# profiles/r01/emit_sweep.md): the first is the default of emit_cuda.
EMIT_VARIANTS = ({"jam": 4, "unroll": 4, "minb": 2}, {"jam": 2, "unroll": 4, "minb": 2},
                 {"jam": 8, "unroll": 2, "minb": 2}, {"jam": 4, "unroll": 4, "minb": 2, "bypass_l1": 0})
SMEM_ACC_BYTES = 192 * 1024   # per-CTA budget for block partials promoted to shared memory
JOIN_COLS = 32                # columns per CTA of a join kernel


class _Emitter:
    def __init__(self, ir: dict, blocks: int, optimize: bool = True, jam: int = JAM,
                 unroll: int = 4, threads: int = CTA_THREADS, minb: int = 2, bypass_l1: int = 1,
                 sync: int = 0, auto: int = 1, cluster: int = 8, cluster_min_bytes: int | None = None,
                 cluster_jam: int = 0, cluster_minb: int = 0, cluster_threads: int = 0):
        self.jam, self.unroll, self.threads, self.minb = int(jam), int(unroll), int(threads), int(minb)
        self.bypass_l1 = bool(bypass_l1)
        self.sync = bool(sync)
        self.auto = bool(auto)         # per-region launch shapes (region_shape) may override the above
        self.ir = ir
        self.st = ir["storage"]
        self.ops = ir["ops"]
        self.blocks = blocks
        self.optimize = optimize
        self.w = _Writer()
        self.scalar_names = {}
        for name, s in self.st.items():
            if s["cls"] == "contracted":
                local = f"{name}_s"
                while local in self.st:
                    local += "_"
                self.scalar_names[name] = local
        self.acc_counter = 0
        # per launch: access table, whether every barrier of the plain scheme is kept,
        # and the block partials that live in shared memory
        self.access: dict = {}
        self.conservative = True
        self.promoted: dict = {}
        self.preloaded: dict = {}      # operand -> register holding it (inside a load/compute batch)
        self.cur_threads = self.threads
        self.strip_axis = None         # set while a region is emitted with a 2-D (block x column strip) grid
        self.row_accs: dict = {}       # row accumulator -> its per-strip partial buffer (strip mode)
        self.tile_axis = None          # set while a region's own slices are dealt out tile by tile
        self.cluster = 0               # cluster size while a region is emitted in cluster mode (else 0)
        self.cluster_size = int(cluster)
        self.cluster_min_bytes = self.CLUSTER_MIN_BYTES if cluster_min_bytes is None else int(cluster_min_bytes)
        self.cluster_jam = int(cluster_jam)      # rows per batch in cluster mode (0: CLUSTER_SHAPE's)
        self.cluster_minb = int(cluster_minb)    # CTAs per SM the registers are sized for (0: CLUSTER_SHAPE's)
        self.cluster_threads = int(cluster_threads)

    # -- names and references (cemit.py:54-110) ----------------------------------
    def index(self, s: dict, block: str | None = None) -> str:
        labs, exts = s["labels"], s["extents"]
        if s["order"] == "scalar":
            core = None
        elif s["order"] == "vec":
            core = labs[0]
        elif s["order"] == "row":
            core = f"{labs[0]} * {exts[1]} + {labs[1]}"
        else:
            core = f"{labs[0]} + {labs[1]} * {exts[0]}"
        if block is None:
            return core or "0"
        size = " * ".join(exts) if exts else "1"
        return block if core is None else f"{block} * ({size}) + {core}"

    def partial_ref(self, name: str, block: str | None) -> str:
        if name in self.promoted:
            return f"{name}_l[{self.st[name]['labels'][0]}]"
        return f"{name}[{self.index(self.st[name], block)}]"

    def ref(self, name: str, block: str | None = None) -> str:
        if name in self.preloaded:
            return self.preloaded[name]
        s = self.st[name]
        if s["cls"] == "contracted":
            return self.scalar_names[name]
        if s["order"] == "scalar":
            if s["cls"] == "input":
                return name                       # by-value kernel parameter
            return f"{name}[0]"                   # scalar output / scalar temp in device memory
        if s["cls"] == "partial":
            return self.partial_ref(name, block)
        return f"{name}[{self.index(s)}]"

    def partial_for(self, result: str) -> str | None:
        for name, s in self.st.items():
            if s["cls"] == "partial" and s["base"] == result:
                return name
        return None

    def target_name(self, op: dict, in_region: bool) -> str:
        if in_region:
            p = self.partial_for(op["result"])
            if p is not None:
                return p
        return op["result"]

    def target(self, op: dict, block: str | None, in_region: bool) -> tuple[str, str]:
        """(C lvalue, storage name) of the op's destination."""
        name = self.target_name(op, in_region)
        if self.st[name]["cls"] == "partial":
            return self.partial_ref(name, block), name
        if self.strip_axis is not None and name in self.row_accs:
            st = self.st[name]
            warps = self.threads // 32
            return (f"{self.row_accs[name]}[((long)blockIdx.y * {warps} + (threadIdx.x >> 5)) * ({st['extents'][0]}) "
                    f"+ {st['labels'][0]}]"), name
        return self.ref(name), name

    def init_lvalue(self, name: str, block: str | None) -> str:
        s = self.st[name]
        if s["cls"] == "contracted":
            return self.scalar_names[name]
        return self.partial_ref(name, block) if s["cls"] == "partial" else self.ref(name)

    def expr(self, op: dict) -> str:
        a = [self.ref(n) for n in op["operands"]]
        if op["kind"] == "copy":
            return a[0]
        sym = {"add": "__dadd_rn", "subtract": "__dsub_rn"}.get(op["kind"], "__dmul_rn")
        return f"{sym}({a[0]}, {a[1]})"           # one rounded op per statement (cemit.py:112-136)

    # -- structure ----------------------------------------------------------------
    @staticmethod
    def is_innermost(loop: dict) -> bool:
        def has_loop(items):
            return any(it["t"] == "loop" or (it["t"] == "par" and has_loop(it["body"]))
                       for it in items)
        return not has_loop(loop["body"])

    def has_sliced_lane_loop(self, items: list) -> bool:
        for it in items:
            if it["t"] == "loop":
                if self.is_innermost(it):
                    if it["sliced"]:
                        return True
                elif self.has_sliced_lane_loop(it["body"]):
                    return True
        return False

    def indexed_by(self, storage_name: str, axis: str) -> bool:
        s = self.st[storage_name]
        return s["cls"] != "contracted" and axis in s["labels"]

    # -- who touches what, and from which threads ---------------------------------------
    # Context of an access: "u0" a uniform statement with a memory target (thread 0 only),
    # "u" a uniform statement executed by every thread, ("l", axis, sliced) a strided loop
    # where thread k owns the elements lo + k, lo + k + blockDim.x, ...
    def analyse(self, items: list, in_region: bool) -> dict:
        table: dict = {}

        def note(name, ctx, mode):
            if self.st[name]["cls"] != "contracted":
                table.setdefault(name, []).append((ctx, mode))

        def stmt(it, lane):
            if it["role"] == "init":
                name = it["target"]
                if lane is None:
                    note(name, "u0", "w")
                else:
                    note(name, lane if self.indexed_by(name, lane[1]) else "u", "w")
                return
            op = self.ops[str(it["op"])]
            tname = self.target_name(op, in_region)
            contracted = self.st[tname]["cls"] == "contracted"
            if lane is None:
                ctx = "u" if contracted else "u0"
                for n in op["operands"]:
                    note(n, ctx, "r")
                note(tname, ctx, "w")
                return
            for n in op["operands"]:
                note(n, lane if self.indexed_by(n, lane[1]) else "u", "r")
            if op["reduction"] and not self.indexed_by(tname, lane[1]):
                note(tname, "u0", "w")            # accumulator: thread 0 adds the CTA sum
            else:
                ctx = lane if self.indexed_by(tname, lane[1]) else "u"
                note(tname, ctx, "w")
                if op["reduction"]:
                    note(tname, ctx, "r")

        def walk(items, lane):
            for it in items:
                if it["t"] == "stmt":
                    stmt(it, lane)
                elif it["t"] == "loop":
                    walk(it["body"], ("l", it["axis"], bool(it["sliced"])) if self.is_innermost(it) else lane)

        walk(items, None)
        return table

    def begin_launch(self, items: list, in_region: bool):
        """Set up barrier policy and shared-memory promotion for one kernel."""
        self.cur_threads = self.threads if in_region else SERIAL_THREADS
        self.access = self.analyse(items, in_region)
        self.promoted = {}
        if not self.optimize:
            self.conservative = True
            return
        # a value written by thread 0 and read by other threads needs the full barrier
        # scheme (write -> barrier -> reads -> barrier -> next write)
        self.conservative = any(
            any(c == "u0" and m == "w" for c, m in acc) and any(c != "u0" and m == "r" for c, m in acc)
            for acc in self.access.values())
        if in_region:
            for name, acc in self.access.items():
                s = self.st[name]
                if s["cls"] == "partial" and s["order"] == "vec" and \
                        all(c == ("l", s["labels"][0], False) for c, _ in acc):
                    self.promoted[name] = s["extents"][0]

    def tile_mappable(self, root: dict) -> bool:
        """A region that is nothing but strided loops over its OWN partition axis (plus uniform
        scalar statements): block p need not be the contiguous slice p -- it can take the tiles
        p, p + blocks, p + 2 blocks, .. of that axis.  All CTAs then sweep the vectors together
        (DRAM pages are shared by neighbouring CTAs) instead of running hundreds of separate
        sequential streams; measured on the hand-written AXPYDOT: 7.0 vs 5.1 TB/s.  Each element
        still has one fixed owner thread, block partials stay deterministic."""
        if not self.optimize or self.conservative:
            return False
        lanes = 0
        for it in root["body"]:
            if it["t"] == "stmt":
                continue
            if it["t"] != "loop" or not self.is_innermost(it) or it["axis"] != root["axis"] or not it["sliced"]:
                return False
            lanes += 1
        return lanes > 0

    # Launch shape of a region that reads a 2-D operand in TWO strided loops of the same outer
    # iteration (ATAX: the row dot, then the row again for the column sums): the second read
    # should come from L2, so the rows in flight (CTAs x jam x row bytes) must fit it -- few,
    # large CTAs and two rows per batch: 296 CTAs x 2 x 64 KiB = 38 MB at N = 8192.
    # B200 sweep (scripts/emit_atax_sweep.py): 0.182 -> 0.120 ms for the max-fuse ATAX at n = 8192.
    REREAD_SHAPE = {"jam": 2, "unroll": 4, "threads": 512, "minb": 2, "bypass_l1": False, "per_sm": 2}

    def rereads(self, items: list) -> bool:
        for it in items:
            if it["t"] != "loop" or self.is_innermost(it):
                continue
            seen = set()
            for inner in it["body"]:
                if inner["t"] == "loop" and self.is_innermost(inner):
                    mats = {n for st in inner["body"] if st["role"] == "compute"
                            for n in self.ops[str(st["op"])]["operands"]
                            if len(self.st[n]["labels"]) == 2 and self.st[n]["cls"] != "contracted"}
                    if mats & seen:
                        return True
                    seen |= mats
            if self.rereads(it["body"]):
                return True
        return False

    def region_shape(self, root: dict):
        """Per-region override of (jam, unroll, threads, minb, bypass_l1) and the CTAs per SM cap;
        None: the emitter's own settings."""
        if self.optimize and self.auto and self.rereads(root["body"]):
            return dict(self.REREAD_SHAPE)
        return None

    def _lane_loops(self, items: list):
        for it in items:
            if it["t"] == "loop":
                if self.is_innermost(it):
                    yield it
                else:
                    yield from self._lane_loops(it["body"])

    # Launch shape of the same kind of region in CLUSTER mode (below): CTA c of a cluster of C does
    # strip c of the strided axis, a batch of `jam` row slices is read from HBM once and a second
    # time from L1 (jam x N / C doubles per CTA), column accumulators are N / C doubles of shared
    # memory whatever N is.
    # B200 sweep at n = 32768 (scripts/emit_cluster_sweep.py, profiles/r02/emit_cluster_sweep.log):
    # ATAX 2.3 -> 5.2 TB/s (0.33 -> 0.73 of the hand-written cluster kernel).
    CLUSTER_SHAPE = {"jam": 4, "unroll": 4, "threads": 256, "minb": 3, "bypass_l1": False, "per_sm": 3}
    # Which variant runs is decided per call from the row length (profiles/r02/emit_cluster_sizes.log,
    # emitted ATAX against the plain mapping): below 80 KiB the plain mapping (0.80-0.87 of the
    # hand-written kernel at n <= 8192), then the smallest cluster whose slice per CTA is at most
    # 40 KiB -- C = 4 at n = 12288 / 16384 (0.88 / 0.79 against 0.76 / 0.62 plain), C = 8 from
    # n = 24576 on (0.94, 0.73 at 32768 against 0.70, 0.33).
    CLUSTER_MIN_BYTES = 80 * 1024
    CLUSTER_SLICE_BYTES = 40 * 1024

    def cluster_mappable(self, root: dict):
        """A region that reads a row twice (`rereads`) needs the whole row between the two reads
        and one accumulator per column: beyond ~16 K columns neither L2 (rows in flight) nor shared
        memory (accumulators) holds that per CTA, and the plain mapping falls to a third of the
        hand-written kernel.  When every strided loop of the region runs over ONE full-extent axis
        other than the partition axis, the C CTAs of a thread-block cluster can split that axis:
        element-wise targets stay owned by one thread of one CTA, sums that leave the axis are
        completed through distributed shared memory (`cluster_allreduce_n`), statements with a
        memory target outside the strided loops are executed by one thread of the cluster.
        Returns the strided axis or None."""
        if not self.optimize or self.conservative or not 2 <= self.cluster_size <= 8:
            return None                                   # (portable cluster sizes only)
        axes = set()

        def walk(its) -> bool:
            for it in its:
                if it["t"] == "stmt":
                    # uniform statement: must not touch anything indexed by a strided axis (checked
                    # once the axis is known, below)
                    continue
                if it["t"] != "loop":
                    return False
                if self.is_innermost(it):
                    if it["sliced"]:
                        return False
                    axes.add(it["axis"])
                    for st in it["body"]:
                        name = st["target"] if st["role"] == "init" else \
                            self.target_name(self.ops[str(st["op"])], True)
                        if it["axis"] in self.st[name]["labels"] and self.st[name]["cls"] != "contracted":
                            continue                      # element-wise in the strided axis
                        if st["role"] != "compute" or not self.ops[str(st["op"])]["reduction"]:
                            return False                  # a plain store that does not move with the axis
                elif not walk(it["body"]):
                    return False
            return True

        if not walk(root["body"]) or len(axes) != 1:
            return None
        v = next(iter(axes))
        if v == root["axis"]:
            return None
        # uniform statements (outside strided loops) must not read or write v-indexed storage
        def uniform_ok(its, in_lane) -> bool:
            for it in its:
                if it["t"] == "loop":
                    if not uniform_ok(it["body"], in_lane or self.is_innermost(it)):
                        return False
                    continue
                if in_lane:
                    continue
                names = [it["target"]] if it["role"] == "init" else \
                    list(self.ops[str(it["op"])]["operands"]) + [self.target_name(self.ops[str(it["op"])], True)]
                if any(self.indexed_by(n, v) for n in names):
                    return False
            return True

        return v if uniform_ok(root["body"], False) else None

    def strip_width(self) -> int:
        return self.threads * self.unroll

    def strip_mappable(self, items: list, part_axis: str | None = None):
        """A region whose statements are all element-wise in ONE full-extent strided axis (no
        uniform statements, no reductions that leave that axis) can be cut into column strips:
        CTA (p, c) does block p of the partition and strip c of the strided axis.  Every CTA then
        holds its column accumulators for one strip only (8 KiB of shared memory instead of 8 N),
        so the SMs are full, and nothing new has to be joined.

        One kind of reduction may leave the axis: a row dot `X[i] += ..` into an output / temporary
        indexed by the partition axis only, which the region otherwise just zeroes (BiCGK's q).
        Its strips write per-strip partials `X_sp_[c][i]`, added up in ascending strip order by a
        small join kernel (`self.row_accs`).  Returns the strided axis or None."""
        self.row_accs = {}
        if not self.optimize or self.conservative:
            return None
        axes = set()
        row_accs = {}

        def row_acc_ok(name: str) -> bool:
            s = self.st[name]
            return (part_axis is not None and s["cls"] in ("output", "temp") and s["order"] == "vec"
                    and s["labels"] == [part_axis])

        def walk(its) -> bool:
            for it in its:
                if it["t"] == "stmt":
                    # the only uniform statement allowed: zeroing a row accumulator
                    if it["role"] == "init" and row_acc_ok(it["target"]):
                        row_accs.setdefault(it["target"], 0)
                        continue
                    return False
                if it["t"] != "loop":
                    return False
                if self.is_innermost(it):
                    if it["sliced"]:
                        return False
                    axes.add(it["axis"])
                    for st in it["body"]:       # every target moves with the strided axis ...
                        name = st["target"] if st["role"] == "init" else \
                            self.target_name(self.ops[str(st["op"])], True)
                        if it["axis"] in self.st[name]["labels"]:
                            continue
                        op = self.ops[str(st["op"])] if st["role"] == "compute" else None
                        if op is None or not op["reduction"] or not row_acc_ok(name):
                            return False
                        row_accs[name] = row_accs.get(name, 0) + 1      # ... or is a row dot
                elif not walk(it["body"]):
                    return False
            return True

        if not walk(items) or len(axes) != 1:
            return None
        for name, count in row_accs.items():
            # exactly one reduction feeds it and nothing in the region reads it
            if count != 1 or any(m == "r" and c != "u0" for c, m in self.access.get(name, ())):
                return None
            if name in {n for it in self._all_stmts(items) if it["role"] == "compute"
                        for n in self.ops[str(it["op"])]["operands"]}:
                return None
        self.row_accs = {name: f"{name}_sp_" for name in row_accs}
        return next(iter(axes))

    def _all_stmts(self, items: list):
        for it in items:
            if it["t"] == "stmt":
                yield it
            else:
                yield from self._all_stmts(it["body"])

    def lane_private(self, name: str, key: tuple) -> bool:
        return all(c == key for c, _ in self.access.get(name, ()))

    def written(self, name: str) -> bool:
        return any(m == "w" for _, m in self.access.get(name, ()))

    def loop_needs_barrier(self, loop: dict, in_region: bool) -> bool:
        """After a strided loop: only when something it touches element-wise is written in
        this launch and also touched with a different thread mapping."""
        if self.conservative:
            return True
        key = ("l", loop["axis"], bool(loop["sliced"]))
        names = set()
        for it in loop["body"]:
            if it["role"] == "init":
                names.add(it["target"])
                continue
            op = self.ops[str(it["op"])]
            names.update(op["operands"])
            tname = self.target_name(op, in_region)
            if not (op["reduction"] and not self.indexed_by(tname, loop["axis"])):
                names.add(tname)
        return any(self.st[n]["cls"] != "contracted" and self.written(n) and not self.lane_private(n, key)
                   for n in names)

    def t0(self) -> str:
        """Guard of a statement with a memory target outside the strided loops: one thread of the
        block -- in cluster mode one thread of the cluster (every CTA holds the same value)."""
        return "threadIdx.x == 0 && c_ == 0" if self.cluster else "threadIdx.x == 0"

    # -- plain emission ------------------------------------------------------------------
    def emit_uniform_stmt(self, stmt: dict, block: str | None, in_region: bool, barrier: bool = True):
        """A statement outside any strided loop: same value in every thread."""
        w = self.w
        barrier = barrier and self.conservative
        if stmt["role"] == "init":
            name = stmt["target"]
            if self.strip_axis is not None and name in self.row_accs:
                return                                   # the strip partial is assigned, not accumulated
            if self.st[name]["cls"] == "contracted":
                w.put(f"{self.scalar_names[name]} = 0.0;")
                return
            w.put(f"if ({self.t0()}) {self.init_lvalue(name, block)} = 0.0;")
            if barrier:
                w.put("__syncthreads();")
            return
        op = self.ops[str(stmt["op"])]
        lhs, sname = self.target(op, block, in_region)
        assign = "+=" if op["reduction"] else "="
        if self.st[sname]["cls"] == "contracted":
            w.put(f"{lhs} {assign} {self.expr(op)};")
        else:
            w.put(f"if ({self.t0()}) {lhs} {assign} {self.expr(op)};")
            if barrier:
                w.put("__syncthreads();")

    def lane_accumulators(self, loop: dict, block: str | None, in_region: bool) -> dict:
        """Reductions whose destination does not move with the strided loop."""
        accs = {}
        for it in loop["body"]:
            if it["t"] == "stmt" and it["role"] == "compute":
                op = self.ops[str(it["op"])]
                if op["reduction"]:
                    lhs, sname = self.target(op, block, in_region)
                    if not self.indexed_by(sname, loop["axis"]):
                        self.acc_counter += 1
                        accs[it["op"]] = (f"lacc{self.acc_counter}", lhs, sname)
        return accs

    def lane_header(self, loop: dict) -> str:
        v = loop["axis"]
        lo, hi = (f"{v}_lo", f"{v}_hi") if loop["sliced"] else ("0", loop["extent"])
        return f"for (long {v} = {lo} + threadIdx.x; {v} < {hi}; {v} += blockDim.x)"

    def is_global_rmw(self, loop: dict, accs: dict, in_region: bool) -> bool:
        for it in loop["body"]:
            if it["role"] == "compute" and it["op"] not in accs:
                op = self.ops[str(it["op"])]
                if op["reduction"] and self.target_name(op, in_region) not in self.promoted:
                    return True
        return False

    def emit_lane_body(self, loop: dict, accs: dict, block: str | None, in_region: bool):
        w = self.w
        for it in loop["body"]:
            if it["role"] == "init":
                w.put(f"{self.init_lvalue(it['target'], block)} = 0.0;")
                continue
            op = self.ops[str(it["op"])]
            if it["op"] in accs:
                w.put(f"{accs[it['op']][0]} += {self.expr(op)};")
                continue
            lhs, _ = self.target(op, block, in_region)
            w.put(f"{lhs} {'+=' if op['reduction'] else '='} {self.expr(op)};")

    def emit_lane_loop(self, loop: dict, block: str | None, in_region: bool):
        """The innermost loop of a nest, strided across the CTA's threads."""
        if self.optimize:
            self.emit_batched_lane(loop, block, in_region, None)
            return
        w = self.w
        accs = self.lane_accumulators(loop, block, in_region)
        for acc, _, _ in accs.values():
            w.put(f"double {acc} = 0.0;")
        # loops that only load, compute and store to their own elements are unrolled so
        # several loads are in flight per thread; loops that read-modify-write global memory
        # are not (measured: unrolling those serialises on the memory dependences, ~10x slower)
        if not self.is_global_rmw(loop, accs, in_region):
            w.put("#pragma unroll 4")
        w.open(self.lane_header(loop))
        self.emit_lane_body(loop, accs, block, in_region)
        w.close()
        for acc, lhs, sname in accs.values():
            w.put(f"{acc} = cta_allreduce({acc}, scratch_);")
            if self.st[sname]["cls"] == "contracted":
                w.put(f"{lhs} += {acc};")
            else:
                w.put(f"if (threadIdx.x == 0) {lhs} += {acc};")
        if self.loop_needs_barrier(loop, in_region):
            w.put("__syncthreads();")

    def streamed_operands(self, loop: dict) -> list:
        """Operands of the strided loop that move with it and are read-only in this launch:
        these are loaded in batches ahead of the arithmetic."""
        names = []
        for it in loop["body"]:
            if it["role"] != "compute":
                continue
            for n in self.ops[str(it["op"])]["operands"]:
                if n not in names and self.indexed_by(n, loop["axis"]) and not self.written(n):
                    names.append(n)
        return names

    def load_of(self, name: str, loop: dict) -> str:
        """Batched load of a read-only operand: 2-D operands pass once (no L1 allocation),
        vectors are reused by the next rows and stay cached."""
        once = len(self.st[name]["labels"]) == 2 and self.bypass_l1
        return f"{'ld_stream' if once else 'ld_keep'}(&{self.ref(name)})"

    def emit_batched_lane(self, loop: dict, block: str | None, in_region: bool, rows):
        """Strided loop as explicit load / compute batches.  `rows` = (axis, scalars) when
        the surrounding loop is jammed: every statement then runs for `jam` rows.

        Per thread and batch: U elements of the strided axis (stride = CTA size, a literal, so
        the compiler sees that they are distinct) times R rows; all loads of the read-only
        operands are issued first, then the statements run in the reference's order (row by
        row for one element, so an element's `+=` chain keeps its ascending-row order)."""
        w = self.w
        v, T = loop["axis"], self.cur_threads
        lo, hi = (f"{v}_lo", f"{v}_hi") if loop["sliced"] else ("0", loop["extent"])
        if self.strip_axis == v and not loop["sliced"]:
            lo, hi = f"{v}_s0_", f"{v}_s1_"               # this CTA's column strip
        accs = self.lane_accumulators(loop, block, in_region)
        R = self.jam if rows else 1
        U = 1 if self.is_global_rmw(loop, accs, in_region) else self.unroll
        a, scalars = rows if rows else (None, [])
        for acc, _, _ in accs.values():
            w.put(f"double {acc}_a[{R}] = {{}};" if rows else f"double {acc} = 0.0;")
        streamed = self.streamed_operands(loop)
        per_row = {n: bool(rows) and a in self.st[n]["labels"] for n in streamed}

        def open_rows(aliases=True):
            if not rows:
                return
            w.put("#pragma unroll")
            w.open(f"for (int r_ = 0; r_ < {R}; ++r_)")
            w.put(f"const long {a} = {a}_b_ + r_; (void){a};")
            if aliases:
                for name in scalars:
                    local = self.scalar_names[name]
                    w.put(f"double &{local} = {local}_a[r_]; (void){local};")
                for acc, _, _ in accs.values():
                    w.put(f"double &{acc} = {acc}_a[r_];")

        def close_rows():
            if rows:
                w.close()

        w.open("")
        tiled = self.tile_axis == v and loop["sliced"]
        if tiled:
            tile = U * T
            w.open(f"for (long t_ = p_; t_ * {tile} < {loop['extent']}; t_ += nblocks_)")
            w.put(f"const long {v}_t0_ = t_ * {tile};")
            w.put(f"const long {v}_t1_ = {v}_t0_ + {tile} < {loop['extent']} ? {v}_t0_ + {tile} : {loop['extent']};")
            lo, hi = f"{v}_t0_", f"{v}_t1_"
        w.put(f"long {v}_b_ = {lo} + threadIdx.x;")
        if U > 1 or streamed:
            w.open(f"for (; {v}_b_ + {(U - 1) * T} < {hi}; {v}_b_ += {U * T})")
            for n in streamed:
                w.put(f"double {n}_v[{R}][{U}];" if per_row[n] else f"double {n}_v[{U}];")
            if streamed:
                w.put("#pragma unroll")
                w.open(f"for (int u_ = 0; u_ < {U}; ++u_)")
                w.put(f"const long {v} = {v}_b_ + u_ * {T};")
                for n in streamed:
                    if not per_row[n]:
                        w.put(f"{n}_v[u_] = {self.load_of(n, loop)};")
                if any(per_row.values()):
                    open_rows(aliases=False)
                    for n in streamed:
                        if per_row[n]:
                            w.put(f"{n}_v[r_][u_] = {self.load_of(n, loop)};")
                    close_rows()
                w.close()
            w.put("#pragma unroll")
            w.open(f"for (int u_ = 0; u_ < {U}; ++u_)")
            w.put(f"const long {v} = {v}_b_ + u_ * {T}; (void){v};")
            open_rows()
            self.preloaded = {n: (f"{n}_v[r_][u_]" if per_row[n] else f"{n}_v[u_]") for n in streamed}
            self.emit_lane_body(loop, accs, block, in_region)
            self.preloaded = {}
            close_rows()
            w.close()
            w.close()
        w.open(f"for (; {v}_b_ < {hi}; {v}_b_ += {T})")           # what is left of the range
        w.put(f"const long {v} = {v}_b_;")
        open_rows()
        self.emit_lane_body(loop, accs, block, in_region)
        close_rows()
        w.close()
        if tiled:
            w.close()
        w.close()
        for acc, lhs, sname in accs.values():
            per_warp = self.strip_axis is not None and sname in self.row_accs
            if per_warp:
                # strip mode: a warp's lanes are summed, lane 0 stores the warp's partial of the
                # row dot; strips x warps partials are added by the row join.  No CTA barrier.
                if rows:
                    w.put(f"warp_reduce_n<{R}>({acc}_a);")
                    open_rows()
                else:
                    w.put(f"{{ double one_[1] = {{{acc}}}; warp_reduce_n<1>(one_); {acc} = one_[0]; }}")
                w.put(f"if ((threadIdx.x & 31) == 0) {lhs} = {acc};")
                close_rows()
                continue
            xbuf = f"xch_ + xpar_ * {self.cluster * self.jam}"
            if rows:
                if self.cluster:
                    w.put(f"cluster_allreduce_n<{R}, {self.cluster}>({acc}_a, scratch_, {xbuf}, xpar_);")
                else:
                    w.put(f"cta_allreduce_n<{R}>({acc}_a, scratch_);")
                open_rows()
            elif self.cluster:
                w.put(f"{{ double one_[1] = {{{acc}}}; cluster_allreduce_n<1, {self.cluster}>(one_, scratch_, {xbuf}, xpar_); "
                      f"{acc} = one_[0]; }}")
            else:
                w.put(f"{acc} = cta_allreduce({acc}, scratch_);")
            if self.st[sname]["cls"] == "contracted":
                w.put(f"{lhs} += {acc};")
            else:
                w.put(f"if ({self.t0()}) {lhs} += {acc};")
            close_rows()
        if self.loop_needs_barrier(loop, in_region):
            w.put("__syncthreads();")

    # -- unroll-and-jam of a loop around strided loops ----------------------------------------
    def jam_legal(self, loop: dict, in_region: bool) -> bool:
        """Iterations of `loop` may be processed JAM at a time when they only meet in
        accumulations: everything written is either private to the iteration (indexed by the
        loop's axis, or a contracted scalar labelled by it) or the target of exactly one
        `+=` statement that nothing else in the body reads."""
        if not self.optimize or self.conservative:
            return False
        a = loop["axis"]
        stmts = []
        lanes = 0
        for it in loop["body"]:
            if it["t"] == "stmt":
                stmts.append(it)
            elif it["t"] == "loop" and self.is_innermost(it) and it["axis"] != a:
                lanes += 1
                stmts.extend(it["body"])
            else:
                return False
        if lanes == 0:
            return False
        reads, shared_writes = set(), {}
        for it in stmts:
            if it["role"] == "init":
                if a not in self.st[it["target"]]["labels"]:
                    return False
                continue
            op = self.ops[str(it["op"])]
            reads.update(op["operands"])
            tname = self.target_name(op, in_region)
            if a in self.st[tname]["labels"]:
                continue
            if self.st[tname]["cls"] == "contracted" or not op["reduction"]:
                return False
            shared_writes[tname] = shared_writes.get(tname, 0) + 1
        return all(n == 1 for n in shared_writes.values()) and not (reads & set(shared_writes))

    def jam_written_scalars(self, loop: dict) -> list:
        names = []
        def visit(items):
            for it in items:
                if it["t"] == "loop":
                    visit(it["body"])
                    continue
                name = it["target"] if it["role"] == "init" else self.ops[str(it["op"])]["result"]
                if self.st[name]["cls"] == "contracted" and name not in names:
                    names.append(name)
        visit(loop["body"])
        return names

    def emit_jammed_loop(self, loop: dict, block: str | None, in_region: bool):
        w = self.w
        a = loop["axis"]
        lo, hi = (f"{a}_lo", f"{a}_hi") if loop["sliced"] else ("0", loop["extent"])
        scalars = self.jam_written_scalars(loop)
        w.open("")                               # scope: the same axis may head several nests
        w.put(f"long {a}_b_ = {lo};")
        w.open(f"for (; {a}_b_ + {self.jam} <= {hi}; {a}_b_ += {self.jam})")
        for name in scalars:
            w.put(f"double {self.scalar_names[name]}_a[{self.jam}];")
        def rows(extra_alias=()):
            """open the per-row loop: row index and the row's private scalars under their usual names"""
            w.put("#pragma unroll")
            w.open(f"for (int r_ = 0; r_ < {self.jam}; ++r_)")
            w.put(f"const long {a} = {a}_b_ + r_; (void){a};")
            for name in scalars:
                local = self.scalar_names[name]
                w.put(f"double &{local} = {local}_a[r_]; (void){local};")
            for acc in extra_alias:
                w.put(f"double &{acc} = {acc}_a[r_];")

        for it in loop["body"]:
            if it["t"] == "stmt":
                rows()
                self.emit_uniform_stmt(it, block, in_region, barrier=False)
                w.close()
            else:
                self.emit_batched_lane(it, block, in_region, (a, scalars))
        w.close()
        # remaining rows one at a time
        w.open(f"for (long {a} = {a}_b_; {a} < {hi}; ++{a})")
        self.emit_items(loop["body"], block, in_region)
        w.close()
        w.close()

    def emit_items(self, items: list, block: str | None, in_region: bool):
        for it in items:
            if it["t"] == "stmt":
                self.emit_uniform_stmt(it, block, in_region)
            elif it["t"] == "loop":
                if self.is_innermost(it):
                    self.emit_lane_loop(it, block, in_region)
                elif self.jam_legal(it, in_region):
                    self.emit_jammed_loop(it, block, in_region)
                else:
                    v = it["axis"]
                    rng = (f"long {v} = {v}_lo; {v} < {v}_hi; ++{v}" if it["sliced"]
                           else f"long {v} = 0; {v} < {it['extent']}; ++{v}")
                    self.w.open(f"for ({rng})")
                    self.emit_items(it["body"], block, in_region)
                    self.w.close()
            else:
                raise ValueError("nested parallel regions are not part of the IR")

    # -- whole translation unit -----------------------------------------------------
    def device_params(self) -> list[tuple[str, str]]:
        """(declaration, name) of everything a kernel may touch, fixed order."""
        out = []
        for name, kind in self.ir["inputs"]:
            out.append((f"double {name}" if kind == "scalar" else f"const double *__restrict__ {name}", name))
        for name, _ in self.ir["outputs"]:
            out.append((f"double *__restrict__ {name}", name))
        for name, s in self.st.items():
            if s["cls"] in ("temp", "partial"):
                out.append((f"double *__restrict__ {name}", name))
        for sp in self.all_row_accs().values():           # per-strip partials of row dots (strip mode)
            out.append((f"double *__restrict__ {sp}", sp))
        out += [(f"long {e}", e) for e in self.ir["extents"]]
        return out

    def all_row_accs(self) -> dict:
        """Row accumulators of every strip-mapped region of the kernel (name -> buffer)."""
        found = {}
        for root in self.ir["roots"]:
            if root["t"] == "par":
                self.begin_launch(root["body"], True)
                if self.strip_mappable(root["body"], root["axis"]) is not None:
                    found.update(self.row_accs)
        self.row_accs = {}
        return found

    def emit_join(self, jname: str, decl: str, pname: str, result: str):
        """Ascending join of the block partials (cemit.py:204-222) as its own kernel."""
        w = self.w
        ps = self.st[pname]
        if not ps["extents"]:
            # scalar: thread k adds blocks k, k + 256, ..; then the fixed-order CTA reduction
            w.open(f"__global__ void __launch_bounds__(256) {jname}({decl}, long nblocks_)")
            w.put("__shared__ double scratch_[32];")
            w.put("double acc = 0.0;")
            w.put(f"for (long b = threadIdx.x; b < nblocks_; b += 256) acc += {pname}[b];")
            w.put("acc = cta_allreduce(acc, scratch_);")
            w.put(f"if (threadIdx.x == 0) {self.ref(result)} = acc;")
            w.close()
            w.put()
            return "1"
        lab, e0 = ps["labels"][0], ps["extents"][0]
        w.open(f"__global__ void __launch_bounds__(256) {jname}({decl}, long nblocks_)")
        # a CTA joins JOIN_COLS adjacent elements: lane = element, warp w adds the w-th
        # eighth of the blocks in 8 independent chains (the partials sit in L2; one dependent
        # chain per element would pay its latency nblocks times); fixed order throughout
        w.put(f"__shared__ double part_[8][{JOIN_COLS}];")
        w.put("const int lane_ = threadIdx.x & 31, warp_ = threadIdx.x >> 5;")
        w.put(f"const long {lab} = (long)blockIdx.x * {JOIN_COLS} + lane_;")
        w.open(f"if ({lab} < {e0})")
        w.put("const long b0_ = (nblocks_ * warp_) / 8, b1_ = (nblocks_ * (warp_ + 1)) / 8;")
        w.put("double a_[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};")
        w.put("long b = b0_;")
        w.open("for (; b + 8 <= b1_; b += 8)")
        w.put("#pragma unroll")
        w.put(f"for (int u = 0; u < 8; ++u) a_[u] += {pname}[(b + u) * ({e0}) + {lab}];")
        w.close()
        w.put("#pragma unroll")
        w.put(f"for (int u = 0; u < 8; ++u) if (b + u < b1_) a_[u] += {pname}[(b + u) * ({e0}) + {lab}];")
        w.put("part_[warp_][lane_] = ((a_[0] + a_[1]) + (a_[2] + a_[3])) + ((a_[4] + a_[5]) + (a_[6] + a_[7]));")
        w.close()
        w.put("__syncthreads();")
        w.open(f"if (warp_ == 0 && {lab} < {e0})")
        w.put(f"{self.ref(result)} = ((part_[0][lane_] + part_[1][lane_]) + (part_[2][lane_] + part_[3][lane_])) + "
              f"((part_[4][lane_] + part_[5][lane_]) + (part_[6][lane_] + part_[7][lane_]));")
        w.close()
        w.close()
        w.put()
        return f"(unsigned)(({e0} + {JOIN_COLS - 1}) / {JOIN_COLS})"

    def emit(self) -> str:
        ir, w = self.ir, self.w
        kname = ir["name"].lower()
        sp_buffers = list(self.all_row_accs().values())
        dparams = self.device_params()
        decl = ", ".join(d for d, _ in dparams)
        call = ", ".join(n for _, n in dparams)
        w.lines.append(f"// {ir['name']}: CUDA emitted for organism {ir['organism'] or '(scalar)'}")
        w.lines.append(_PRELUDE)

        launches = []          # host-side launch statements
        regions = 0
        serial_group: list = []
        uses_smem = False

        def scalars_decl():
            for local in self.scalar_names.values():
                w.put(f"double {local} = 0.0;")
            w.put(f"__shared__ double scratch_[{32 * self.jam}];")
            w.put("(void)scratch_;")

        def flush_serial():
            nonlocal regions
            if not serial_group:
                return
            fname = f"{kname}_serial{regions}"
            regions += 1
            self.begin_launch(serial_group, False)
            w.open(f"__global__ void __launch_bounds__({SERIAL_THREADS}) {fname}({decl})")
            scalars_decl()
            self.emit_items(serial_group, None, False)
            w.close()
            w.put()
            launches.append(f"{fname}<<<1, {SERIAL_THREADS}, 0, 0>>>({call});")
            serial_group.clear()

        for root in ir["roots"]:
            if root["t"] != "par":
                serial_group.append(root)
                continue
            flush_serial()
            org_t = int(ir["threads"][root["slot"]])
            t = max(org_t, self.blocks)
            base_name = f"{kname}_region{regions}"
            nb = f"nb{regions}_"
            regions += 1
            ax, ext = root["axis"], root["extent"]
            saved = (self.jam, self.unroll, self.threads, self.minb, self.bypass_l1)
            launches.append(f"long {nb} = 0;")

            def variant(cluster_axis, C=0):
                """One kernel for the region (plain / strips, or cluster mode) and the host statements
                that size and launch it; `nb` receives its block count."""
                nonlocal uses_smem
                out = []
                fname = base_name + (f"c{C}" if cluster_axis else "")
                shape = dict(self.CLUSTER_SHAPE) if cluster_axis else self.region_shape(root)
                if cluster_axis and self.cluster_jam:
                    shape["jam"] = self.cluster_jam
                if cluster_axis and self.cluster_minb:
                    shape["minb"] = self.cluster_minb
                if cluster_axis and self.cluster_threads:
                    shape["threads"] = self.cluster_threads
                if shape:
                    self.jam, self.unroll, self.threads = shape["jam"], shape["unroll"], shape["threads"]
                    self.minb, self.bypass_l1 = shape["minb"], shape["bypass_l1"]
                self.begin_launch(root["body"], True)
                # When the strided (innermost) loops run over the block's own slice, a
                # slice narrower than the CTA leaves threads idle: cap the block count
                # so every CTA gets at least a CTA-width of the axis (never below the
                # organism's own count).  Any count is legal for the block formula.
                tiles = self.tile_mappable(root) and not cluster_axis
                if tiles:
                    # interleaved tiles: as many blocks as there are tiles at most
                    tile = self.unroll * self.threads
                    out.append(f"{nb} = ({root['extent']} + {tile - 1}) / {tile}; "
                               f"if ({nb} < {org_t}) {nb} = {org_t}; if ({nb} > {t}) {nb} = {t};")
                elif self.has_sliced_lane_loop(root["body"]):
                    out.append(f"{nb} = {root['extent']} / {self.threads}; "
                               f"if ({nb} < {org_t}) {nb} = {org_t}; if ({nb} > {t}) {nb} = {t};")
                else:
                    out.append(f"{nb} = {t};")
                if shape and not C:
                    uses_smem = True                     # (sms_ is read from the device below)
                    out.append(f"{{ long cap_ = (long)sms_ * {shape['per_sm']}; if (cap_ < {org_t}) cap_ = {org_t}; "
                               f"if ({nb} > cap_) {nb} = cap_; }}")
                smem_args = ""
                strip = None if cluster_axis else self.strip_mappable(root["body"], root["axis"])
                strip_ext = None
                if strip is not None:
                    # 2-D grid: blockIdx.x = block of the partition, blockIdx.y = column strip
                    strip_ext = next(l["extent"] for l in self._lane_loops(root["body"]))
                    sw = self.strip_width()
                    out.append(f"const long strips{regions}_ = ({strip_ext} + {sw - 1}) / {sw};")
                    out.append(f"{{ long want_ = ((long)sms_ * 8 + strips{regions}_ - 1) / strips{regions}_; "
                               f"if (want_ < {org_t}) want_ = {org_t}; if ({nb} > want_) {nb} = want_; }}")
                    uses_smem = True                     # (sms_ is read from the device below)
                    for name, sp in self.row_accs.items():
                        e0 = self.st[name]["extents"][0]
                        out.append(f"{{ const size_t need_ = sizeof(double) * (size_t)strips{regions}_ * {self.threads // 32} * (size_t){e0}; "
                                   f"if (need_ > {sp}_n_) {{ if ({sp}_c_) cudaFreeAsync({sp}_c_, 0); cudaMallocAsync(&{sp}_c_, need_, 0); {sp}_n_ = need_; }} "
                                   f"{sp} = {sp}_c_; }}")
                if cluster_axis:
                    # the cluster's C CTAs split the strided axis: strip c = [c sw, (c + 1) sw)
                    strip_ext = next(l["extent"] for l in self._lane_loops(root["body"]))
                    out.append(f"const long csw{regions}_ = ((({strip_ext} + {C - 1}) / {C}) + 1) & ~1L;")
                if self.promoted and strip is not None:
                    total = len(self.promoted) * self.strip_width()
                    out.append(f"const size_t smb{regions}_ = sizeof(double) * {total};")
                    out.append(f"const int sm_ok{regions}_ = 1;")
                    smem_args = f", sm_ok{regions}_"
                elif self.promoted and cluster_axis:
                    out.append(f"const size_t smb{regions}_ = sizeof(double) * {len(self.promoted)} * (size_t)csw{regions}_;")
                    out.append(f"const int sm_ok{regions}_ = smb{regions}_ <= {SMEM_ACC_BYTES // 2};")
                    out.append(f"static bool attr{regions}_ = false; if (!attr{regions}_) {{ cudaFuncSetAttribute({fname}, "
                               f"cudaFuncAttributeMaxDynamicSharedMemorySize, {SMEM_ACC_BYTES // 2}); attr{regions}_ = true; }}")
                    smem_args = f", sm_ok{regions}_"
                elif self.promoted:
                    # block partials indexed by the strided axis only: each thread owns its
                    # elements for the whole launch, so they accumulate in shared memory and
                    # reach the partial buffer once, at the end (when they fit; else in place)
                    uses_smem = True
                    total = " + ".join(f"(size_t){e}" for e in self.promoted.values())
                    out.append(f"const size_t smb{regions}_ = sizeof(double) * ({total});")
                    out.append(f"const int sm_ok{regions}_ = smb{regions}_ <= {SMEM_ACC_BYTES};")
                    out.append(f"if (sm_ok{regions}_) {{ long fit_ = (long)sms_ * (long)((227 * 1024) / (smb{regions}_ + 2048)); "
                               f"if (fit_ < {org_t}) fit_ = {org_t}; if ({nb} > fit_) {nb} = fit_; }}")
                    out.append(f"static bool attr{regions}_ = false; if (!attr{regions}_) {{ cudaFuncSetAttribute({fname}, "
                               f"cudaFuncAttributeMaxDynamicSharedMemorySize, {SMEM_ACC_BYTES}); attr{regions}_ = true; }}")
                    smem_args = f", sm_ok{regions}_"
                if cluster_axis:
                    # one wave: as many clusters as the device holds at once (clusters live inside a
                    # GPC, so this is less than SMs x CTAs per SM / C), asked once per footprint
                    dynb = f"(sm_ok{regions}_ ? smb{regions}_ : 0)" if self.promoted else "0"
                    out.append("cudaLaunchConfig_t cfg_ = {}; cudaLaunchAttribute cattr_;")
                    out.append(f"cattr_.id = cudaLaunchAttributeClusterDimension; cattr_.val.clusterDim.x = {C}; "
                               "cattr_.val.clusterDim.y = 1; cattr_.val.clusterDim.z = 1;")
                    out.append(f"cfg_.blockDim = dim3({self.threads}); cfg_.dynamicSmemBytes = {dynb}; cfg_.stream = 0; "
                               "cfg_.attrs = &cattr_; cfg_.numAttrs = 1;")
                    out.append(f"static size_t occ_for{regions}_ = ~(size_t)0; static int occ{regions}_ = 0;")
                    out.append(f"if (occ_for{regions}_ != cfg_.dynamicSmemBytes) {{ cfg_.gridDim = dim3({C} * 64); "
                               f"if (cudaOccupancyMaxActiveClusters(&occ{regions}_, {fname}, &cfg_) != cudaSuccess || occ{regions}_ < 1) "
                               f"occ{regions}_ = 1; occ_for{regions}_ = cfg_.dynamicSmemBytes; }}")
                    out.append(f"{{ long cap_ = occ{regions}_; if (cap_ < {org_t}) cap_ = {org_t}; if ({nb} > cap_) {nb} = cap_; }}")
                # min-blocks in the launch bounds: without it ptxas aims for full occupancy, keeps the
                # register count low and sinks every batched load down to its use
                bounds = f"{self.threads}, {self.minb}" if self.optimize else f"{self.threads}"
                w.open(f"__global__ void __launch_bounds__({bounds}) {fname}({decl}, long nblocks_"
                       + (", int sm_ok_" if self.promoted else "") + (", long csw_" if C else "") + ")")
                scalars_decl()
                if C:
                    w.put(f"__shared__ double xch_[{2 * C * max(self.jam, 1)}];")
                    w.put("int xpar_ = 0; (void)xpar_;")
                    w.put(f"const long p_ = blockIdx.x / {C};")
                    w.put(f"const long c_ = blockIdx.x % {C}; (void)c_;")
                else:
                    w.put("const long p_ = blockIdx.x;")
                w.put(f"const long {ax}_lo = ({ext} * p_) / nblocks_;")
                w.put(f"const long {ax}_hi = ({ext} * (p_ + 1)) / nblocks_;")
                w.put(f"(void){ax}_lo; (void){ax}_hi;")
                self.tile_axis = root["axis"] if tiles else None
                if strip is not None:
                    sw = self.strip_width()
                    w.put(f"const long {strip}_s0_ = (long)blockIdx.y * {sw};")
                    w.put(f"const long {strip}_s1_ = {strip}_s0_ + {sw} < {strip_ext} ? {strip}_s0_ + {sw} : {strip_ext};")
                    self.strip_axis = strip
                if cluster_axis:
                    cv = cluster_axis
                    w.put(f"const long {cv}_s0_ = c_ * csw_ < {strip_ext} ? c_ * csw_ : {strip_ext};")
                    w.put(f"const long {cv}_s1_ = {cv}_s0_ + csw_ < {strip_ext} ? {cv}_s0_ + csw_ : {strip_ext};")
                    self.strip_axis = cv
                    self.cluster = C
                if self.promoted:
                    w.put("extern __shared__ double dyn_[];")
                    offset = "0"
                    for name, e in self.promoted.items():
                        size = self.st[name]["extents"][0]
                        if strip is not None:          # X_l[j] is valid for the strip's j
                            w.put(f"double *{name}_l = dyn_ + ({offset}) - {strip}_s0_; (void)sm_ok_;")
                            offset += f" + {self.strip_width()}"
                        elif cluster_axis:
                            w.put(f"double *{name}_l = sm_ok_ ? dyn_ + ({offset}) - {cluster_axis}_s0_ : {name} + p_ * ({size});")
                            offset += " + csw_"
                        else:
                            w.put(f"double *{name}_l = sm_ok_ ? dyn_ + ({offset}) : {name} + p_ * ({size});")
                            offset += f" + {e}"
                self.emit_items(root["body"], "p_", True)
                if self.promoted:
                    w.open("if (sm_ok_)")
                    for name in self.promoted:
                        s = self.st[name]
                        lab, size = s["labels"][0], s["extents"][0]
                        sa = strip if strip is not None else cluster_axis
                        lo, hi = (f"{sa}_s0_", f"{sa}_s1_") if sa is not None else ("0", size)
                        w.put(f"for (long {lab} = {lo} + threadIdx.x; {lab} < {hi}; {lab} += blockDim.x) "
                              f"{name}[p_ * ({size}) + {lab}] = {name}_l[{lab}];")
                    w.close()
                if C:
                    # nobody leaves while a peer may still read its exchange buffer
                    w.put('asm volatile("barrier.cluster.arrive.release.aligned;\\n\\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");')
                self.strip_axis = None
                self.tile_axis = None
                self.cluster = 0
                w.close()
                w.put()
                dyn = f"sm_ok{regions}_ ? smb{regions}_ : 0" if self.promoted else "0"
                if strip is not None:
                    grid = f"dim3((unsigned){nb}, (unsigned)strips{regions}_)"
                elif C:
                    grid = f"(unsigned)({nb} * {C})"
                else:
                    grid = f"(unsigned){nb}"
                if C:
                    out.append(f"cfg_.gridDim = dim3({grid});")
                    out.append(f"cudaLaunchKernelEx(&cfg_, {fname}, {call}, {nb}{smem_args}, csw{regions}_);")
                else:
                    out.append(f"{fname}<<<{grid}, {self.threads}, {dyn}, 0>>>({call}, {nb}{smem_args});")
                for name, sp in (self.row_accs.items() if strip is not None else ()):
                    # ascending (strip, warp) partials, a thread per row
                    e0, lab = self.st[name]["extents"][0], self.st[name]["labels"][0]
                    jname = f"{kname}_rows{regions}_{name}"
                    w.open(f"__global__ void __launch_bounds__(256) {jname}({decl}, long strips_)")
                    w.put(f"const long {lab} = (long)blockIdx.x * 256 + threadIdx.x;")
                    w.open(f"if ({lab} < {e0})")
                    w.put(f"double acc = {sp}[{lab}];")
                    w.put(f"for (long c = 1; c < strips_; ++c) acc += {sp}[c * ({e0}) + {lab}];")
                    w.put(f"{self.ref(name)} = acc;")
                    w.close()
                    w.close()
                    w.put()
                    out.append(f"{jname}<<<(unsigned)(({e0} + 255) / 256), 256, 0, 0>>>({call}, strips{regions}_ * {self.threads // 32});")
                self.row_accs = {}
                self.promoted = {}
                self.jam, self.unroll, self.threads, self.minb, self.bypass_l1 = saved
                return out

            cl_axis = None
            if self.optimize and self.auto and self.cluster_size and self.rereads(root["body"]):
                self.begin_launch(root["body"], True)
                # (a region that can be cut into independent column strips -- the two reads of a row do
                #  not depend on each other, BiCGK's two products -- is better off that way: measured)
                if self.strip_mappable(root["body"], root["axis"]) is None:
                    cl_axis = self.cluster_mappable(root)
                self.row_accs = {}
            plain = variant(None)
            if cl_axis is not None:
                sizes = [c for c in (4, 8) if c <= self.cluster_size] or [self.cluster_size]
                row_ext = next(l["extent"] for l in self._lane_loops(root["body"]))
                launches.append(f"const size_t row{regions}_ = (size_t){row_ext} * sizeof(double);")
                for k, C in enumerate(sizes):
                    cond = f"row{regions}_ >= {self.cluster_min_bytes}"
                    if k + 1 < len(sizes):
                        cond += f" && row{regions}_ <= {C * self.CLUSTER_SLICE_BYTES}"
                    clustered = variant(cl_axis, C)
                    launches.append(("if" if k == 0 else "} else if") + f" ({cond}) {{")
                    launches.extend("    " + st for st in clustered)
                launches.append("} else {")
                launches.extend("    " + st for st in plain)
                launches.append("}")
            else:
                launches.extend(plain)
            for result in root["partials"]:
                pname = self.partial_for(result)
                jname = f"{kname}_join{regions}_{result}"
                grid = self.emit_join(jname, decl, pname, result)
                launches.append(f"{jname}<<<{grid}, 256, 0, 0>>>({call}, {nb});")
        flush_serial()

        # host entry point: the reference's signature (cemit.py:225-241), device pointers
        hparams = []
        for name, kind in ir["inputs"]:
            hparams.append(f"double {name}" if kind == "scalar" else f"const double *{name}")
        for name, _ in ir["outputs"]:
            hparams.append(f"double *{name}")
        hparams += [f"long {e}" for e in ir["extents"]]
        w.open(f'extern "C" void {kname}({", ".join(hparams)})')
        if uses_smem:
            w.put("static int sms_ = 0;")
            w.open("if (!sms_)")
            w.put("int dev_ = 0; cudaGetDevice(&dev_);")
            w.put("cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev_);")
            w.close()
        temps = []
        for name, s in self.st.items():
            if s["cls"] == "temp":
                size = " * ".join(f"(size_t){e}" for e in s["extents"]) if s["extents"] else "1"
                temps.append((name, size))
            elif s["cls"] == "partial":
                region = next(r for r in ir["roots"] if r["t"] == "par" and s["base"] in r["partials"])
                t = max(int(ir["threads"][region["slot"]]), self.blocks)
                size = " * ".join([f"(size_t){t}"] + [f"(size_t){e}" for e in s["extents"]])
                temps.append((name, size))
        if temps:
            # keep freed temporaries in the stream-ordered pool across calls (the default
            # release threshold of 0 hands them back to the driver at every sync)
            w.put("static bool pool_ready_ = false;")
            w.open("if (!pool_ready_)")
            w.put("int dev_ = 0; cudaGetDevice(&dev_);")
            w.put("cudaMemPool_t pool_; cudaDeviceGetDefaultMemPool(&pool_, dev_);")
            w.put("unsigned long long keep_ = ~0ULL;")
            w.put("cudaMemPoolSetAttribute(pool_, cudaMemPoolAttrReleaseThreshold, &keep_);")
            w.put("pool_ready_ = true;")
            w.close()
        cached = self.optimize and (temps or sp_buffers)
        if cached:
            # Temporaries and partial buffers are kept from call to call, per HOST THREAD and device,
            # and only ever grow: no allocation on the steady-state path (the reference mallocs and
            # frees per call, cemit.py:183-202; two calls from two threads still get buffers of their
            # own, so "thread-safe per output buffer", holds).  Launches are on stream 0,
            # so the next call's kernels are ordered after this call's.
            w.put("static thread_local int cache_dev_ = -1;")
            w.put("int dev_now_ = 0; cudaGetDevice(&dev_now_);")
            names = [n for n, _ in temps] + list(sp_buffers)
            for n in names:
                w.put(f"static thread_local double *{n}_c_ = nullptr; static thread_local size_t {n}_n_ = 0;")
            w.put("if (dev_now_ != cache_dev_) { " + " ".join(f"{n}_c_ = nullptr; {n}_n_ = 0;" for n in names)
                  + " cache_dev_ = dev_now_; }")
        for name, size in temps:
            if cached:
                w.put(f"{{ const size_t need_ = sizeof(double) * ({size}); if (need_ > {name}_n_) {{ "
                      f"if ({name}_c_) cudaFreeAsync({name}_c_, 0); cudaMallocAsync(&{name}_c_, need_, 0); {name}_n_ = need_; }} }}")
                w.put(f"double *{name} = {name}_c_;")
            else:
                w.put(f"double *{name} = nullptr;")
                w.put(f"cudaMallocAsync(&{name}, sizeof(double) * ({size}), 0);")
        for sp in sp_buffers:
            w.put(f"double *{sp} = nullptr;")
        for stmt in launches:
            w.put(stmt)
        if not cached:
            for name, _ in temps:      # stream-ordered pool: no device-wide sync per temporary
                w.put(f"cudaFreeAsync({name}, 0);")
        if self.sync or not self.optimize:
            w.put("cudaStreamSynchronize(0);")       # the reference's protocol: results ready on return
        # (default: stream-ordered like the library's own device-pointer entry points -- operands
        #  are device buffers, temporaries are freed in stream order; the caller synchronises)
        w.close()
        w.put()
        w.open(f'extern "C" int {kname}_last_cuda_error(void)')
        w.put("return (int)cudaGetLastError();")
        w.close()
        return "\n".join(w.lines) + "\n"


def emit_cuda(ir: dict, blocks: int = DEFAULT_BLOCKS, optimize: bool = True, **tune) -> GeneratedKernel:
    """Render a loop-IR snapshot as a standalone CUDA translation unit.
    Deterministic: the same IR, `blocks` and `optimize` always yield byte-identical source.
    `optimize=False` prints the plain mapping only (every barrier, no unroll-and-jam, block
    partials accumulated in global memory).  `tune`: jam (rows per batch), unroll (of the
    strided loop under a batch), threads (per CTA of a parallel region), minb (CTAs per SM the
    register budget is sized for), sync (1: cudaStreamSynchronize before returning), cluster (CTAs per
    cluster of the cluster-mode variant of regions that read a row twice, 0: none), cluster_min_bytes
    (row length from which that variant runs; 0 forces it), cluster_jam, bypass_l1 (0: 2-D operands are loaded L1-allocating; ATAX-like
    bodies that read a row twice gain 10 %)."""
    em = _Emitter(ir, int(blocks), bool(optimize), **tune)
    source = em.emit()
    params = []
    for name, kind in ir["inputs"]:
        params.append((f"double {name}" if kind == "scalar" else f"const double *{name}", name))
    for name, _ in ir["outputs"]:
        params.append((f"double *{name}", name))
    params += [(f"long {e}", e) for e in ir["extents"]]
    return GeneratedKernel(source=source, kernel_name=ir["name"].lower(), params=tuple(params),
                           organism_key=ir["organism"], threads=tuple(ir["threads"]))


# ---------------------------------------------------------------------------
# toolchain (runtime.py:26-83, with nvcc and the -fPIC translation)

DEFAULT_TEMPLATE = "{cc} -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a {src} -o {bin}"


@dataclass
class NvccToolchain:
    """`cache_dir` (or $BTO_NVCC_CACHE): compiled translation units are kept there under the hash of
    (source, command), so a search that meets the same organism and launch shape again -- or a
    second process -- skips nvcc (3-5 s per kernel)."""
    cc: str | None = None
    template: str = ""
    cache_dir: str | None = None

    def __post_init__(self):
        if not self.cc:
            self.cc = os.environ.get("BTO_NVCC") or shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
        if not self.template:
            self.template = os.environ.get("BTO_NVCC_TEMPLATE", DEFAULT_TEMPLATE)
        if self.cache_dir is None:
            self.cache_dir = os.environ.get("BTO_NVCC_CACHE") or None

    @property
    def available(self) -> bool:
        return bool(self.cc) and (shutil.which(self.cc) is not None or Path(self.cc).exists())

    def compile(self, source: str, workdir, name: str = "kernel", shared: bool = True) -> Path:
        if not self.available:
            raise ToolchainError("nvcc not found (set BTO_NVCC)")
        workdir = Path(workdir)
        src = workdir / f"{name}.cu"
        src.write_text(source)
        binary = workdir / (f"{name}.so" if shared else name)
        cmd = shlex.split(self.template.format(cc=self.cc, src=src, bin=binary))
        if shared:       # nvcc does not take -fPIC directly
            cmd += ["-shared", "-Xcompiler", "-fPIC"]
        cached = None
        if self.cache_dir:
            import hashlib
            key = hashlib.sha256((source + "\0" + self.template + "\0" + str(shared)).encode()).hexdigest()[:32]
            cached = Path(self.cache_dir) / (key + (".so" if shared else ".bin"))
            if cached.exists():
                shutil.copyfile(cached, binary)
                if not shared:
                    binary.chmod(0o755)
                return binary
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise ToolchainError(f"compile failed ({' '.join(cmd)}):\n{proc.stderr.strip()}")
        if cached is not None:
            cached.parent.mkdir(parents=True, exist_ok=True)
            tmp = cached.with_suffix(cached.suffix + f".{os.getpid()}.tmp")
            shutil.copyfile(binary, tmp)
            os.replace(tmp, cached)                  # atomic: concurrent searches may share the cache
        return binary


def run_emitted(binary, kernel: GeneratedKernel, ir: dict, inputs: dict, extents: dict) -> dict:
    """Call an emitted kernel (run_kernel's protocol, runtime.py:99-150): numpy or
    torch CUDA inputs; outputs NaN-prefilled; returns the outputs dict."""
    import numpy as np
    import torch

    lib = ctypes.CDLL(str(binary))
    fn = getattr(lib, kernel.kernel_name)
    fn.restype = None
    st = ir["storage"]
    on_gpu = any(hasattr(inputs.get(n), "is_cuda") and inputs[n].is_cuda for n, _ in ir["inputs"])
    args, keep, outs = [], [], {}
    for name, kind in ir["inputs"]:
        if kind == "scalar":
            args.append(ctypes.c_double(float(inputs[name])))
            continue
        want = tuple(int(extents[e]) for e in st[name]["extents"])
        v = inputs[name]
        t = v if hasattr(v, "is_cuda") else torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float64)))
        if tuple(t.shape) != want:
            raise ValueError(f"{name}: expected shape {want}, got {tuple(t.shape)}")
        t = t.to("cuda", torch.float64)
        if st[name]["order"] == "col":
            t = t.t()
        t = t.contiguous()
        keep.append(t)
        args.append(ctypes.c_void_p(t.data_ptr()))
    for name, kind in ir["outputs"]:
        size = 1
        for e in st[name]["extents"]:
            size *= int(extents[e])
        buf = torch.full((size,), float("nan"), dtype=torch.float64, device="cuda")
        outs[name] = buf
        args.append(ctypes.c_void_p(buf.data_ptr()))
    args += [ctypes.c_long(int(extents[e])) for e in ir["extents"]]
    torch.cuda.synchronize()
    fn(*args)
    err = getattr(lib, kernel.kernel_name + "_last_cuda_error")()
    torch.cuda.synchronize()
    if err:
        raise ToolchainError(f"emitted kernel failed with CUDA error {err}")
    result = {}
    for name, kind in ir["outputs"]:
        buf = outs[name]
        if kind == "scalar":
            result[name] = float(buf[0])
            continue
        shape = tuple(int(extents[e]) for e in st[name]["extents"])
        if st[name]["order"] == "col":
            val = buf.reshape(shape[::-1]).t().contiguous()
        else:
            val = buf.reshape(shape)
        result[name] = val if on_gpu else val.cpu().numpy()
    return result


def time_emitted(binary, kernel: GeneratedKernel, ir: dict, dev_inputs: dict, extents: dict,
                 reps: int = 5) -> float:
    """Best-of-`reps` seconds of the emitted entry point alone (its launches, joins,
    temporaries and final sync) on device-resident operands, outputs preallocated."""
    import math

    import torch

    lib = ctypes.CDLL(str(binary))
    fn = getattr(lib, kernel.kernel_name)
    fn.restype = None
    st = ir["storage"]
    args, keep = [], []
    for name, kind in ir["inputs"]:
        if kind == "scalar":
            args.append(ctypes.c_double(float(dev_inputs[name])))
            continue
        t = dev_inputs[name]
        if st[name]["order"] == "col":
            t = t.t()
        t = t.contiguous()
        keep.append(t)
        args.append(ctypes.c_void_p(t.data_ptr()))
    for name, kind in ir["outputs"]:
        size = 1
        for e in st[name]["extents"]:
            size *= int(extents[e])
        buf = torch.empty((size,), dtype=torch.float64, device="cuda")
        keep.append(buf)
        args.append(ctypes.c_void_p(buf.data_ptr()))
    args += [ctypes.c_long(int(extents[e])) for e in ir["extents"]]
    torch.cuda.synchronize()
    fn(*args)                                                      # warm-up
    best = math.inf
    for _ in range(reps):
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        fn(*args)
        stop.record()
        stop.synchronize()
        best = min(best, start.elapsed_time(stop) * 1e-3)
    if getattr(lib, kernel.kernel_name + "_last_cuda_error")():
        raise ToolchainError("emitted kernel failed while being timed")
    return best


# ---------------------------------------------------------------------------
# fused execution of specs outside the hand-written set (mixed orientations, non-corpus kernels)

_EMITTED: dict = {}           # GeneratedKernel.source -> (shared object, emitted kernel, IR)
_EMITTED_BY_SPEC: dict = {}   # .bto text -> handle (the search and the compile run once per spec and process)
NOMINAL_EXTENT = 4096         # organisms are ranked by the analytic model at this size (where it is fitted)


def ir_for_spec(ref_graph, extents: dict | None = None, generations: int = 20, seed: int = 0) -> dict:
    """Loop IR of the organism the REFERENCE's own search (MFGA, search.py:834) finds best for
    `ref_graph` under the organism-level GPU cost model (`AnalyticOrganismCost`), max-fuse being one
    of the candidates.  Needs the reference importable (it is, where this package is a drop-in)."""
    from matfuse import SearchConfig, cached, contract_arrays, lower, max_fuse, run_strategy
    names = tuple(ref_graph.extent_names)
    # (a kernel of vectors only is priced at the element count of a NOMINAL_EXTENT-square matrix)
    ext = extents or {e: (NOMINAL_EXTENT * NOMINAL_EXTENT if len(names) == 1 else NOMINAL_EXTENT) for e in names}
    fitness = cached(AnalyticOrganismCost(ref_graph, ext))
    best = max_fuse(ref_graph, 8)
    best_cost = fitness(best).total
    try:
        res = run_strategy("mfga", ref_graph, SearchConfig(core_count=8, generations=generations, seed=seed), fitness)
        if res.best is not None and res.best_fitness < best_cost:
            best = res.best
    except Exception:                               # a search that fails leaves max-fuse
        pass
    return ir_from_matfuse(contract_arrays(lower(best, ref_graph)))


def emitted_kernel_for(graph, toolchain: "NvccToolchain | None" = None, ir: dict | None = None):
    """A FUSED kernel for a spec the hand-written sequences do not cover: the reference lowers the
    organism its search picks (`ir_for_spec`), `emit_cuda` prints it, nvcc compiles it once (cached
    by source hash).  `graph`: this package's TypedSpec / KernelSpec or the reference's
    DataflowGraph.  Returns a GeneratedKernel whose `source` is "emitted:<shared object>", or None
    when the reference or nvcc is not available (the caller falls back to the unfused executor).
    `ir`: a stored snapshot instead of the search (machines without the reference)."""
    import tempfile
    tc = toolchain or NvccToolchain(cache_dir=os.environ.get("BTO_NVCC_CACHE") or
                                    str(Path(tempfile.gettempdir()) / "bto_b200_emit"))
    if not tc.available:
        return None
    memo_key = None
    if ir is None and toolchain is None and not (hasattr(graph, "data") and hasattr(graph, "ops")):
        from .spec import format_kernel
        memo_key = format_kernel(graph.spec if hasattr(graph, "spec") else graph)
        if memo_key in _EMITTED_BY_SPEC:
            return _EMITTED_BY_SPEC[memo_key]
    if ir is None:
        try:
            import matfuse                              # noqa: F401
            from matfuse.graph import build_dataflow, infer_types
        except ImportError:
            return None
        if hasattr(graph, "data") and hasattr(graph, "ops"):
            ref_graph = graph                           # the reference's own DataflowGraph
        else:
            from .spec import format_kernel
            spec = graph.spec if hasattr(graph, "spec") else graph
            ref_graph = infer_types(build_dataflow(matfuse.parse_kernel(format_kernel(spec))))
        ir = ir_for_spec(ref_graph)
    kernel = emit_cuda(ir)
    work = Path(tempfile.mkdtemp(prefix="bto-emit-"))
    path = tc.compile(kernel.source, work, name=kernel.kernel_name)
    handle = GeneratedKernel(source=f"emitted:{path}", kernel_name=kernel.kernel_name, params=kernel.params,
                             organism_key=kernel.organism_key, threads=kernel.threads)
    _EMITTED[handle.source] = (path, kernel, ir)
    if memo_key is not None:
        _EMITTED_BY_SPEC[memo_key] = handle
    return handle


def emitted_entry(source: str):
    """(shared object, emitted kernel, IR) behind an "emitted:..." handle."""
    try:
        return _EMITTED[source]
    except KeyError:
        raise ToolchainError(f"{source} was not produced by emitted_kernel_for in this process") from None


# ---------------------------------------------------------------------------
# empirical fitness for organisms (cost.py:124-208 with a GPU back end)

def measure_empirical_ir(ir: dict, graph, extents: dict, reps: int = 5,
                         validate_extents: dict | None = None, blocks: int = DEFAULT_BLOCKS,
                         toolchain: NvccToolchain | None = None, source_filter=None,
                         tolerance: float = 1e-10, optimize: bool = True, variants=None):
    """Emit, compile, validate, then time one lowered organism; +inf with the
    reference's diagnostics on any failure (cost.py:176-207).  `graph` is this
    package's TypedSpec of the same kernel; validation compares against the
    independent spec evaluator (cost.evaluate_spec).  `source_filter` is the
    reference's fault-injection hook (cost.py:148,186).  `variants`: launch-shape settings
    (dicts of emit_cuda's tunables, e.g. EMIT_VARIANTS) to try after the default one has
    validated; the best time is reported."""
    import math

    import torch

    from .cost import CostReport, evaluate_spec
    from .runtime import gen_inputs, max_rel_error, workdir

    def failure(kind: str, detail: str) -> CostReport:
        return CostReport(total=math.inf, source="empirical", diagnostic=f"{kind}: {detail}")

    kernel = emit_cuda(ir, blocks=blocks, optimize=optimize)
    source = source_filter(kernel.source) if source_filter is not None else kernel.source
    try:
        lib = (toolchain or NvccToolchain()).compile(source, workdir(), name="kernel", shared=True)
    except ToolchainError as exc:
        return failure("compile-failure", str(exc))
    vext = validate_extents or {k: min(64, v) for k, v in extents.items()}
    try:
        inputs = gen_inputs(graph, vext, seed=7)
        dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in inputs.items()}
        got = run_emitted(lib, kernel, ir, dev, vext)
        want = evaluate_spec(graph.spec, dev)
    except Exception as exc:  # noqa: BLE001 -- a crash is a fitness failure, not an error
        return failure("runtime-crash", repr(exc))
    err = max_rel_error({k: (v if isinstance(v, float) else v.cpu().numpy()) for k, v in got.items()},
                        {k: (v if isinstance(v, float) else v.cpu().numpy()) for k, v in want.items()})
    if not err < tolerance:
        return failure("numerical-mismatch", f"max relative error {err:.3e}")
    try:
        inputs = gen_inputs(graph, extents, seed=7)
        dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v) for k, v in inputs.items()}
        best = time_emitted(lib, kernel, ir, dev, extents, reps=reps)
        for idx, tune in enumerate(variants or ()):
            alt = emit_cuda(ir, blocks=blocks, optimize=optimize, **tune)
            if alt.source == kernel.source:
                continue
            alt_lib = (toolchain or NvccToolchain()).compile(alt.source, workdir(), name=f"kernel_v{idx}",
                                                             shared=True)
            best = min(best, time_emitted(alt_lib, alt, ir, dev, extents, reps=reps))
    except Exception as exc:  # noqa: BLE001
        return failure("runtime-crash", repr(exc))
    return CostReport(total=best, source="empirical")


class OrganismTimer:
    """Drop-in for the reference's `EmpiricalTimer` (cost.py:124-160) where both the
    reference and a GPU are present: `fitness(organism) -> CostReport` through
    lower -> contract_arrays -> CUDA emission -> nvcc -> validate -> CUDA events.
    Usable directly with `matfuse.search.run_strategy`."""

    parallel_safe = False

    def __init__(self, ref_graph, extents: dict | None = None, reps: int = 5,
                 validate_extents: dict | None = None, blocks: int = DEFAULT_BLOCKS,
                 source_filter=None, optimize: bool = True, variants=None):
        from .runtime import _convert_expr
        from .spec import Decl, KernelSpec, infer_shapes
        spec = ref_graph.spec
        self.ref_graph = ref_graph
        self.graph = infer_shapes(KernelSpec(
            spec.name,
            tuple((n, Decl(d.kind, d.orientation)) for n, d in spec.inputs),
            tuple((n, Decl(d.kind, d.orientation)) for n, d in spec.outputs),
            tuple((s.target, _convert_expr(s.value)) for s in spec.statements)))
        self.extents = extents or {n: 1000 for n in ref_graph.extent_names}
        self.reps, self.validate_extents, self.blocks = reps, validate_extents, blocks
        self.source_filter = source_filter
        self.optimize, self.variants = optimize, variants

    def key_salt(self) -> str:
        return ("empirical-cuda:" if self.optimize else "empirical-cuda-plain:") + ",".join(f"{k}={v}" for k, v in sorted(self.extents.items()))

    def __call__(self, organism):
        from matfuse import contract_arrays, lower
        ir = ir_from_matfuse(contract_arrays(lower(organism, self.ref_graph)))
        return measure_empirical_ir(ir, self.graph, self.extents, self.reps,
                                    validate_extents=self.validate_extents, blocks=self.blocks,
                                    source_filter=self.source_filter, optimize=self.optimize,
                                    variants=self.variants)


# ---------------------------------------------------------------------------
# analytic fitness for organisms: HBM bytes, occupancy and barrier steps of the
# kernels `emit_cuda` would print (the organism-level half of the GPU cost model)

@dataclass(frozen=True)
class EmitModel:
    """Coefficients of `estimate_cost_ir`, fitted on the 360 timings of
    profiles/r01/organism_times.json (120 organisms x n = 1024, 2048, 4096) by
    scripts/fit_emit_model.py."""
    peak_gbs: float = 6500.0        # HBM ceiling of a full grid
    cta_gbs: float = 97.5          # what one CTA streams on its own
    launch_us: float = 6.0         # per kernel launch (incl. its share of the final sync)
    step_us: float = 0.50           # one strided-loop execution that ends in a barrier / CTA reduction
    free_step_us: float = 0.0       # ... that ends in neither (barrier analysis removed them)
    trip_us: float = 0.17           # one trip of a thread through a strided loop
    jam_trip_us: float = 0.30       # the same per row when rows are batched (unroll-and-jam; a trip then
                                    # carries `unroll` elements per row, hence the larger figure)
    rmw_trip_us: float = 0.14       # a trip that read-modify-writes global memory
    stmt_us: float = 0.84           # a uniform statement that writes memory and needs its barrier
    free_stmt_us: float = 0.07      # ... and does not
    alloc_us: float = 0.01           # stream-ordered malloc + free of one temporary / partial per call
                                    # (the reference pays malloc/free per call too, cemit.py:183-202)
    sm_count: int = 148


def estimate_cost_ir(ir: dict, extents: dict, model: EmitModel | None = None,
                     blocks: int = DEFAULT_BLOCKS):
    """Deterministic seconds estimate of the CUDA `emit_cuda(ir, blocks)` prints.

    Per launch: time = launch + max(bytes / bandwidth(blocks), steps), where
    * bytes   -- every 2-D operand streams once per execution of the strided loop
                 that touches it (no cache between loop nests on a GPU: re-reads
                 count, unlike cost.py:80-86); vectors indexed by the strided
                 axis stay cache-resident per CTA and count once per block;
    * bandwidth grows with the number of CTAs up to the HBM ceiling (a serial
      root runs in ONE CTA -- the GPU analogue of an unpartitioned CPU loop;
      shared-memory accumulators cap the CTAs per SM);
    * steps   -- the longest block's chain of strided-loop executions (barriers,
                 CTA reductions, read-modify-write trips) and uniform memory
                 writes, which bounds latency-dominated organisms.  The emitter's own
                 decisions are asked for, not guessed: whether a loop is jammed, which
                 barriers its analysis removes, which partials live in shared memory.
    Returns cost.CostReport(source="analytic")."""
    from .cost import CostReport

    m = model or EmitModel()
    st, ops = ir["storage"], ir["ops"]
    ext = {k: float(v) for k, v in extents.items()}
    per_launch = []
    launches = 0
    em = _Emitter(ir, blocks)

    def has_loop(items):
        return any(it["t"] == "loop" for it in items)

    # 2-D (block x column strip) mapping of the launch; `width` = columns of a strip.  (The cluster
    # variants the emitter adds for rows of 80 KiB and more are not modelled: the coefficients are
    # fitted at n <= 4096, where they never run.)
    strip = {"axis": None, "count": 1.0, "width": 0.0, "reread_free": False}

    def walk(items, trips, nb, threads, acc, in_region, batch, seen=None):
        """acc: dict(bytes=, steps=) for one launch; `trips` executions per block, `batch`
        rows handled per execution (1 unless the enclosing loop is jammed)."""
        seen = set() if seen is None else seen
        for it in items:
            if it["t"] == "stmt":
                target = it["target"] if it["role"] == "init" else ops[str(it["op"])]["result"]
                if st[target]["cls"] != "contracted":
                    acc["steps"] += trips * batch * (m.stmt_us if em.conservative else m.free_stmt_us)
                continue
            rng = ext[it["extent"]] / nb if it["sliced"] else ext[it["extent"]]
            if has_loop(it["body"]):
                jam = em.jam if em.jam_legal(it, in_region) else 1
                walk(it["body"], trips * max(rng / jam, 1.0), nb, threads, acc, in_region, jam, set())
                continue
            # strided (innermost) loop
            ctas = nb
            if strip["axis"] == it["axis"] and not it["sliced"]:
                rng = min(rng, strip["width"])                 # a CTA walks one strip of it
                ctas = nb * strip["count"]
            per_thread = max(1.0, rng / threads)
            mats, vecs, rmw = set(), set(), False
            accs = em.lane_accumulators(it, "p_" if in_region else None, in_region)
            for s in it["body"]:
                if s["role"] == "init":
                    names = [s["target"]]
                else:
                    op = ops[str(s["op"])]
                    names = list(op["operands"]) + [op["result"]]
                for n in names:
                    s_ = st[n]
                    if s_["cls"] == "contracted" or it["axis"] not in s_["labels"]:
                        continue
                    (mats if len(s_["labels"]) == 2 else vecs).add(n)
            rmw = em.is_global_rmw(it, accs, in_region)
            if strip["reread_free"]:
                mats, _ = mats - seen, seen.update(mats)
            acc["bytes"] += 8.0 * len(mats) * rng * trips * batch * ctas + 8.0 * len(vecs) * rng * ctas
            ends_in_sync = bool(accs) or em.loop_needs_barrier(it, in_region)
            trip = m.rmw_trip_us if rmw else (m.jam_trip_us if batch > 1 else m.trip_us)
            acc["steps"] += trips * ((m.step_us if ends_in_sync else m.free_step_us) + per_thread * batch * trip)

    def close(acc, nb):
        bw = min(m.peak_gbs, m.cta_gbs * min(nb, 4 * m.sm_count)) * 1e9
        per_launch.append((m.launch_us + max(acc["bytes"] / bw * 1e6, acc["steps"])) * 1e-6)

    serial_items, serial = [], None

    def flush_serial():
        nonlocal serial, launches
        if not serial_items:
            return
        em.begin_launch(serial_items, False)
        serial = {"bytes": 0.0, "steps": 0.0}
        walk(serial_items, 1.0, 1.0, float(SERIAL_THREADS), serial, False, 1)
        close(serial, 1.0)
        launches += 1
        serial_items.clear()

    for root in ir["roots"]:
        if root["t"] != "par":
            serial_items.append(root)
            continue
        flush_serial()
        org_t = float(ir["threads"][root["slot"]])
        nb = max(org_t, float(blocks))
        saved = (em.jam, em.unroll, em.threads, em.minb, em.bypass_l1)
        shape = em.region_shape(root)
        if shape:                                     # the emitter's per-region launch shape
            em.jam, em.unroll, em.threads = shape["jam"], shape["unroll"], shape["threads"]
            nb = min(nb, max(org_t, float(m.sm_count * shape["per_sm"])))
        em.begin_launch(root["body"], True)
        if em.has_sliced_lane_loop(root["body"]):
            nb = min(nb, max(org_t, float(int(ext[root["extent"]]) // em.threads)))
        axis = em.strip_mappable(root["body"], root["axis"])
        row_joins = len(em.row_accs)
        strip["axis"], strip["count"], strip["width"], strip["reread_free"] = axis, 1.0, float(em.strip_width()), False
        if axis is not None:
            width = ext[next(l["extent"] for l in em._lane_loops(root["body"]))]
            strip["count"] = float(-(-int(width) // em.strip_width()))
            nb = min(nb, max(org_t, float(-(-m.sm_count * 8 // int(strip["count"])))))
        elif em.promoted:
            smem = 8.0 * sum(ext[e] for e in em.promoted.values())
            if smem <= SMEM_ACC_BYTES:
                nb = min(nb, max(org_t, m.sm_count * float(int(227 * 1024 // (smem + 2048)))))
            else:
                em.promoted = {}                       # too long: they stay in the partial buffer
        nb = max(1.0, min(nb, ext[root["extent"]]))
        acc = {"bytes": 0.0, "steps": 0.0}
        walk(root["body"], 1.0, nb, float(em.threads), acc, True, 1)
        close(acc, nb * strip["count"])
        for _ in range(row_joins if axis is not None else 0):    # join of a row dot's strip partials
            per_launch.append((m.launch_us + 8.0 * ext[root["extent"]] * (strip["count"] + 1)
                               / (m.peak_gbs * 1e9) * 1e6) * 1e-6)
            launches += 1
        strip.update(axis=None, count=1.0, reread_free=False)
        em.row_accs = {}
        em.jam, em.unroll, em.threads, em.minb, em.bypass_l1 = saved
        launches += 1
        for result in root["partials"]:          # join: read nb partial rows, write the result
            p = st[em.partial_for(result)]
            size = 1.0
            for e in p["extents"]:
                size *= ext[e]
            per_launch.append((m.launch_us + 8.0 * size * (nb + 1) / (m.peak_gbs * 1e9) * 1e6) * 1e-6)
            launches += 1
    flush_serial()
    nalloc = sum(1 for s in st.values() if s["cls"] in ("temp", "partial"))
    per_launch.append(nalloc * m.alloc_us * 1e-6)
    contracted = tuple(sorted(n for n, s in st.items() if s["cls"] == "contracted"))
    return CostReport(total=float(sum(per_launch)), source="analytic", per_root=tuple(per_launch),
                      contracted=contracted, partition_nodes=launches)


class AnalyticOrganismCost:
    """Fitness callable over the reference's Organism objects (cost.py:106-121 with
    the GPU model): organism -> lower -> contract_arrays -> estimate_cost_ir."""

    parallel_safe = True

    def __init__(self, ref_graph, extents: dict, model: EmitModel | None = None,
                 blocks: int = DEFAULT_BLOCKS):
        self.ref_graph, self.extents, self.model, self.blocks = ref_graph, dict(extents), model, blocks

    def key_salt(self) -> str:
        return "analytic-cuda:" + ",".join(f"{k}={v}" for k, v in sorted(self.extents.items()))

    def __call__(self, organism):
        from matfuse import contract_arrays, lower
        ir = ir_from_matfuse(contract_arrays(lower(organism, self.ref_graph)))
        return estimate_cost_ir(ir, self.extents, self.model, self.blocks)
