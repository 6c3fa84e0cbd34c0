"""Fitness functions for the GPU path: HBM-bytes/occupancy model and CUDA-event timer.

Replaces the two fitness plug-ins of the reference (`cost.py`):

* `estimate_cost` / `AnalyticGpuCost`  <->  `estimate_cost` / `AnalyticCost`
  (cost.py:64-121).  The reference prices an organism by streamed array
  elements divided by threads plus a fixed overhead per partition node; it
  knows nothing about caches.  The GPU model prices a launch VARIANT of a
  fused sequence by the bytes that actually cross HBM -- algorithmic traffic,
  the write + re-read of every materialised intermediate (which the
  reference's distinct-array rule does not count: GEMVER's B, cost.py:80-86),
  and the cross-CTA partial buffers -- divided by the bandwidth the launch
  geometry can sustain (Little's law on bytes in flight per SM, capped by the
  measured read or read+write HBM ceiling), plus a latency term per kernel
  launch and per collective.
* `GpuEmpiricalTimer`  <->  `EmpiricalTimer` / `measure_empirical`
  (cost.py:124-208): validate first (a wrong-answer variant never gets a finite
  fitness), then time with CUDA events on the launch stream: 1 warm-up, min of
  `reps`.  Failures map to `CostReport(total=inf, diagnostic="<kind>: ...")`
  with the reference's kinds (`runtime-crash`, `numerical-mismatch`;
  `compile-failure` when the library is missing).
* `FitnessMemo` / `cached`  <->  cost.py:211-241 (own memo table; `CachedFitness` is an alias).

A variant is what the GPU search explores instead of an organism: the kernel
plus the launch tunables of include/bto_b200.h section 4.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from . import _native
from .spec import TypedSpec, match_corpus

__all__ = [
    "CostReport", "GpuMachineModel", "GpuVariant", "Traffic", "hbm_traffic",
    "estimate_cost", "AnalyticGpuCost", "GpuEmpiricalTimer", "measure_empirical",
    "CachedFitness", "FitnessMemo", "cached", "validation_extents", "variant_space", "evaluate_spec",
]


@dataclass(frozen=True)
class CostReport:
    """Same fields as the reference's (cost.py:50-61)."""
    total: float                      # seconds (both sources, unlike the reference)
    source: str                       # "analytic" | "empirical"
    per_root: tuple[float, ...] = ()  # seconds per kernel launch of the sequence
    contracted: tuple[str, ...] = ()  # intermediates that never reach HBM
    partition_nodes: int = 0          # kernel launches
    diagnostic: str | None = None

    @property
    def failed(self) -> bool:
        return math.isinf(self.total)


@dataclass(frozen=True)
class GpuMachineModel:
    """B200 as the model sees it.  Bandwidths are the measured ceilings of this
    pool (profiles/r01): pure-read kernels top out near 7.15 TB/s, read+write
    streams at the driver-measured copy figure."""
    sm_count: int = 148
    read_gbs: float = 7150.0
    copy_gbs: float = 6551.0
    latency_us: float = 0.75            # HBM latency under load (Little's law)
    duty: float = 0.28                  # share of a CTA's life its loads are in flight when
                                        # every unit ends in a row reduction + barrier
                                        # (calibrated on the 1-CTA/SM rows of
                                        # profiles/r01/sweep1_first.json)
    duty_stream: float = 0.6            # same for passes without row dots (T, T+rank-2)
    launch_us: float = 2.5              # back-to-back launch gap + ramp per kernel
    collective_us: float = 25.0         # small NCCL all-reduce over NVLink
    regs_per_sm: int = 65536
    max_threads_per_sm: int = 2048
    bytes_per_scalar: float = 8.0
    extents: tuple[tuple[str, int], ...] = (("M", 32768), ("N", 32768))

    def extent(self, name: str) -> int:
        for key, val in self.extents:
            if key == name:
                return val
        raise KeyError(f"extent {name!r} not bound")


@dataclass(frozen=True)
class GpuVariant:
    """A launch variant of one fused sequence: the GPU search point."""
    kernel: str
    tuning: tuple[tuple[str, int], ...] = ()

    def key(self) -> str:
        return self.kernel + "{" + ",".join(f"{k}={v}" for k, v in sorted(self.tuning)) + "}"

    def get(self, name: str, default: int = 0) -> int:
        return dict(self.tuning).get(name, default)


# per-pass defaults of csrc/api.cu (mv_default): rows, vec, CTAs/SM, min blocks
_PASS_DEFAULT = {"NT": (8, 1, 8, 4), "NN": (8, 1, 4, 4), "TR": (16, 1, 2, 1),
                 "T": (32, 1, 2, 1), "N": (8, 2, 8, 2)}
# registers per thread of the shipped instantiations (nvcc -Xptxas -v)
_PASS_REGS = {"NT": 64, "NN": 64, "TR": 180, "T": 128, "N": 64}
# passes of each sequence: (kind, matrices read, matrices written)
_SEQUENCE = {
    "bicgk": [("NT", 1, 0)], "gesummv": [("NN", 2, 0)], "dgemv": [("N", 1, 0)],
    "gemver": [("TR", 1, 1), ("N", 1, 0)], "dgemvt": [("T", 1, 0), ("N", 1, 0)],
    "atax2": [("N", 1, 0), ("T", 1, 0)], "atax": [("ATAX", 1, 0)],
}
_CONTRACTED = {"axpydot": ("t0",), "vadd": ("t0",), "waxpby": ("t0", "t1"),
               "atax": ("t0",), "batax": ("t0", "t1"), "gesummv": ("t0", "t1", "t2", "t3"),
               "dgemv": ("t0", "t1", "t2"), "gemver": ("t0", "t1", "t2", "t4"),
               "dgemvt": ("t1",), "bicgk": ()}


@dataclass(frozen=True)
class Traffic:
    algorithmic: float                 # SURVEY.md 8d minimum
    rereads: float = 0.0               # matrix passes beyond the minimum
    partials: float = 0.0              # cross-CTA partial buffers, written + read
    launches: int = 1
    passes: tuple = field(default_factory=tuple)   # (kind, read B, write B, bytes in flight/SM)

    @property
    def total(self) -> float:
        return self.algorithmic + self.rereads + self.partials


def _pass_geometry(kind: str, variant: GpuVariant, machine: GpuMachineModel, M: int, N: int):
    rows, vec, per_sm, minb = _PASS_DEFAULT[kind]
    rows = variant.get("mv_rows") or rows
    vec = variant.get("mv_vec") or vec
    per_sm = variant.get("grid_per_sm") or per_sm
    minb = variant.get("mv_minb") or minb
    regs = max(32, min(255, machine.regs_per_sm // (256 * minb))) if variant.get("mv_minb") \
        else _PASS_REGS[kind]
    resident = max(1, min(machine.regs_per_sm // (256 * regs), machine.max_threads_per_sm // 256,
                          per_sm))
    strip = 512 * vec
    nstrips = -(-N // strip)
    units = -(-M // rows) * nstrips
    grid = max(1, min(machine.sm_count * per_sm, -(-units // 4)))    # >= 4 units per CTA
    slots = min(grid, -(-grid // nstrips) + 1)
    matrices = 2 if kind == "NN" else 1
    inflight = resident * 256 * rows * vec * 16 * matrices     # bytes in flight per SM
    return nstrips, slots, inflight


# Co-resident clusters of the single-pass ATAX kernel on a 148-SM B200 (clusters live inside a GPC;
# profiles/r02/cluster_probe.log) -- what cudaOccupancyMaxActiveClusters answers the library.
ATAX_CLUSTERS_148 = {1: 148, 2: 74, 3: 45, 4: 33, 5: 26, 6: 22, 7: 15, 8: 15, 9: 15, 10: 11, 16: 7}


def atax_cluster_choice(N: int, sm_count: int = 148) -> tuple[int, int, int, int]:
    """(cluster size, KMAX, rows per panel, co-resident clusters) the library picks for a row of N
    columns: the restatement of csrc/host_sequences.cuh::plan_atax -- every built size priced as
    (1150 / TR + 62.5 KMAX) / clusters, ties to the larger SM coverage."""
    best = None
    for c, ncl148 in ATAX_CLUSTERS_148.items():
        w = -(-N // c)
        w += w & 1
        if -(-w // 16) * 16 * (c - 1) < N:
            w = -(-w // 16) * 16
        if c > 1 and (c - 1) * w >= N:
            continue
        kmax = -(-w // 512)
        if kmax > 8:
            kmax = 1 << (kmax - 1).bit_length()
        if kmax > 16 or (kmax == 16 and c < 16):
            continue
        if c in (3, 5, 6, 7, 10) and not 5 <= kmax <= 8:
            continue                                  # the wide-slice sizes are built for 5..8 iterations
        tr = 8 if kmax <= 2 else 4 if kmax <= 4 else 2 if kmax <= 8 else 1
        ncl = max(1, ncl148 * sm_count // 148)
        cost = (1150.0 / tr + 62.5 * kmax) / ncl
        if best is None or cost < best[0] * 0.999 or (cost < best[0] * 1.001 and ncl * c > best[4] * best[1]):
            best = (cost, c, kmax, tr, ncl)
    if best is None:
        raise ValueError(f"no cluster size holds a row of {N} columns")
    return best[1], best[2], best[3], best[4]


def hbm_traffic(kernel: str, M: int, N: int, variant: GpuVariant | None = None,
                machine: GpuMachineModel | None = None) -> Traffic:
    """Bytes crossing HBM for one call of `kernel` under `variant`."""
    variant = variant or GpuVariant(kernel)
    machine = machine or GpuMachineModel()
    kernel = kernel.lower()
    algo = _native.bytes_min(kernel, M, N)
    if kernel in ("axpydot", "vadd", "waxpby"):
        per_sm = 2048 * 16 * 3 * max(1, variant.get("vec_unroll", 2)) // 2
        wr = 8.0 * M
        return Traffic(algo, 0.0, 0.0, 1, (("V", algo - wr, wr, per_sm),))
    seq = kernel
    if kernel in ("atax", "batax"):
        fused = variant.get("atax_fused", 1) and N % 2 == 0 and N <= 16 * 8192
        seq = "atax" if fused else "atax2"
    passes, partials, rereads = [], 0.0, 0.0
    joins = 0
    if kernel in ("atax", "batax") and N <= 512 and variant.get("skinny", 1):
        # shared-row kernel (csrc/skinny_kernels.cuh): single pass, one partial row per CTA
        grid = machine.sm_count * (variant.get("grid_per_sm") or 4)
        return Traffic(algo, 0.0, 2 * 8.0 * grid * N, 2, (("N", 8.0 * M * N, 0.0, 128 * 1024),))
    for idx, (kind, reads, writes) in enumerate(_SEQUENCE[seq]):
        if kind == "ATAX":
            c = variant.get("atax_cluster")
            if c:
                clusters = max(1, ATAX_CLUSTERS_148.get(c, machine.sm_count // c) * machine.sm_count // 148)
            else:
                c, _, _, clusters = atax_cluster_choice(N, machine.sm_count)
            partials += 2 * 8.0 * clusters * N
            passes.append((kind, 8.0 * M * N, 0.0, 64 * 1024))
            continue
        nstrips, slots, inflight = _pass_geometry(kind, variant, machine, M, N)
        if N <= 512 and variant.get("skinny", 1):
            # shared-row kernels: row results written in-kernel, one partial row per CTA for T
            if "T" in kind:
                partials += 2 * 8.0 * machine.sm_count * (variant.get("grid_per_sm") or 4) * N
                joins += 1
        elif kind == "NN" and (N >= 4096 or N <= 2048) and M >= 4 * machine.sm_count and variant.get("rowstream", 1):
            pass                        # whole-row streaming (csrc/rowstream_kernels.cuh): no partials, no join
        else:
            if "N" in kind:
                partials += 2 * 8.0 * nstrips * M * (2 if kind == "NN" else 1)
            if "T" in kind:
                partials += 2 * 8.0 * slots * N
            joins += 1
        passes.append((kind, 8.0 * M * N * reads, 8.0 * M * N * writes, inflight))
        if seq == "atax2" and idx == 1:
            rereads += 8.0 * M * N
    joins += sum(1 for k, *_ in passes if k == "ATAX")
    return Traffic(algo, rereads, partials, len(passes) + joins, tuple(passes))


def estimate_cost(variant: GpuVariant, graph, machine: GpuMachineModel) -> CostReport:
    """Deterministic seconds estimate of one variant: a pure function of its inputs."""
    M = machine.extent("M")
    N = machine.extent("N") if "N" in dict(machine.extents) else 1
    traffic = hbm_traffic(variant.kernel, M, N, variant, machine)
    per_launch = []
    small = (traffic.total - sum(p[1] + p[2] for p in traffic.passes)) / max(1, len(traffic.passes))
    for kind, rd, wr, inflight in traffic.passes:
        ceiling = machine.copy_gbs if wr > 0.1 * rd else machine.read_gbs
        if kind in ("ATAX", "V"):
            duty = 1.0                                   # TMA ring / pure streaming
        else:
            duty = machine.duty if "N" in kind else machine.duty_stream
        littles = duty * inflight * machine.sm_count / (machine.latency_us * 1e-6) / 1e9
        bw = min(ceiling, littles) * 1e9
        per_launch.append((rd + wr + small) / bw + machine.launch_us * 1e-6)
    joins = traffic.launches - len(traffic.passes)
    per_launch += [machine.launch_us * 1e-6] * joins
    world = variant.get("world", 1)
    if world > 1 and variant.kernel not in ("gesummv", "dgemv", "vadd", "waxpby"):
        per_launch.append(machine.collective_us * 1e-6)
    return CostReport(total=float(sum(per_launch)), source="analytic",
                      per_root=tuple(per_launch),
                      contracted=_CONTRACTED.get(variant.kernel, ()),
                      partition_nodes=traffic.launches)


class AnalyticGpuCost:
    """Fitness callable backed by estimate_cost; safe to share across threads."""

    parallel_safe = True

    def __init__(self, graph, machine: GpuMachineModel):
        self.graph, self.machine = graph, machine

    def key_salt(self) -> str:
        return "analytic-gpu:" + ",".join(f"{k}={v}" for k, v in self.machine.extents)

    def __call__(self, variant: GpuVariant) -> CostReport:
        return estimate_cost(variant, self.graph, self.machine)


# ---------------------------------------------------------------------------
# validate-before-time

def evaluate_spec(spec, inputs: dict) -> dict:
    """Evaluate the kernel statements as written with torch fp64 ops on the
    inputs' device -- the role interp.reference_evaluate plays for the
    reference's timer (cost.py:199): a checker that shares no code with the
    hand-written kernels."""
    import torch

    env = {}
    for name, decl in spec.inputs:
        value = inputs[name]
        if decl.kind == "scalar":
            env[name] = ("scalar", float(value))
        elif decl.kind == "vector":
            env[name] = ("col" if decl.orientation == "column" else "row", value)
        else:
            env[name] = ("mat", value)

    def ev(e):
        if e[0] == "var":
            return env[e[1]]
        if e[0] == "t":
            kind, data = ev(e[1])
            return {"col": "row", "row": "col", "mat": "mat"}[kind], \
                (data.t() if kind == "mat" else data)
        (lk, ld), (rk, rd) = ev(e[1]), ev(e[2])
        if e[0] in "+-":
            return lk, (ld + rd if e[0] == "+" else ld - rd)
        if lk == "scalar" or rk == "scalar":
            return (rk, ld * rd) if lk == "scalar" else (lk, ld * rd)
        if lk == "row" and rk == "col":
            return "scalar", float(torch.dot(ld, rd))
        if lk == "col" and rk == "row":
            return "mat", torch.outer(ld, rd)
        if lk == "mat" and rk == "col":
            return "col", torch.mv(ld, rd)
        raise ValueError(f"cannot multiply {lk} by {rk}")

    for target, expr in spec.statements:
        env[target] = ev(expr)
    return {name: env[name][1] for name, _ in spec.outputs}


#: elements of the largest operand up to which the timed extents themselves are validated
_VALIDATE_FULL_BELOW = 1 << 26


def validation_extents(extents: dict) -> dict:
    """Extents at which a variant is checked before it is timed.

    The reference validates at min(64, extent) (cost.py:199-202) because its generated loops are
    the same code at every size.  Here the dispatch depends on the shape: narrow matrices take the
    shared-row kernels, the cluster size of ATAX follows N, whole-row streaming needs N >= 4096,
    and a 64 x 64 problem never enters the unrolled paths -- so a 64-extent check would validate
    kernels the timed run never launches.  Validation therefore runs at the timed extents when
    they are small enough for the in-product evaluator (`evaluate_spec` builds matrix-sized
    temporaries), else at the same N with fewer rows: every dispatch decision of the library is
    made on N and on M >= a few thousand rows, and `measure_empirical` additionally compares
    the launch signatures of the two runs."""
    ext = {k: int(v) for k, v in extents.items()}
    size = 1
    for v in ext.values():
        size *= v
    if size <= _VALIDATE_FULL_BELOW or "N" not in ext or "M" not in ext:
        return ext
    rows = max(4096, _VALIDATE_FULL_BELOW // max(1, ext["N"]))
    ext["M"] = min(ext["M"], rows)
    return ext


def measure_empirical(variant: GpuVariant, graph: TypedSpec, extents: dict, reps: int = 5,
                      validate_extents: dict | None = None, fault=None,
                      tolerance: float = 1e-10) -> CostReport:
    """Validate, then time one variant; +inf with a diagnostic on any failure.

    `fault` is the test hook standing where the reference's `source_filter`
    stands (cost.py:148,186): a callable applied to the outputs dict before
    validation, used to prove wrong answers never receive a finite fitness."""
    import torch
    from .runtime import gen_inputs, gpu_kernel, max_rel_error, run_kernel_async

    def failure(kind: str, detail: str) -> CostReport:
        return CostReport(total=math.inf, source="empirical", diagnostic=f"{kind}: {detail}")

    try:
        _native.load()
        kernel = gpu_kernel(graph)
    except (_native.NativeLibraryMissing, NotImplementedError) as exc:
        return failure("compile-failure", str(exc))
    saved = {k: _native.get_tuning(k) for k, _ in variant.tuning}
    try:
        try:
            _native.set_tuning(**dict(variant.tuning))
        except _native.BtoError as exc:
            return failure("compile-failure", str(exc))
        vext = validate_extents or validation_extents(extents)

        def alloc(ext, seed):
            host = gen_inputs(graph, ext, seed=seed)
            dev = {k: (torch.from_numpy(v).cuda() if hasattr(v, "shape") else v)
                   for k, v in host.items()}
            outs = {}
            for name, decl in graph.spec.outputs:
                size = 1
                for d in graph.dims[name]:
                    size *= int(ext[d])
                outs[name] = torch.full((size,), float("nan"), dtype=torch.float64, device="cuda")
            return dev, outs

        try:
            dev, outs = alloc(vext, 7)
            run_kernel_async(kernel, graph, dev, vext, outs)
            validated_dispatch = _native.launch_signature()
            torch.cuda.synchronize()
            got = {n: (float(outs[n][0]) if d.kind == "scalar" else
                       outs[n].reshape(tuple(int(vext[x]) for x in graph.dims[n])).cpu().numpy())
                   for n, d in graph.spec.outputs}
            if fault is not None:
                got = fault(got)
            want = evaluate_spec(graph.spec, dev)
            want = {n: (v if isinstance(v, float) else v.cpu().numpy()) for n, v in want.items()}
        except Exception as exc:
            return failure("runtime-crash", repr(exc))
        err = max_rel_error(got, want)
        if not err < tolerance:
            return failure("numerical-mismatch", f"max relative error {err:.3e}")
        try:
            del dev, outs
            dev, outs = alloc(extents, 7)
            run_kernel_async(kernel, graph, dev, extents, outs)       # warm-up, untimed
            if validate_extents is None and _native.launch_signature() != validated_dispatch:
                # the kernels about to be timed are not the ones that were checked
                return failure("validation-mismatch",
                               f"extents {vext} validated a different kernel dispatch than {extents} runs")
            best = math.inf
            stream = torch.cuda.current_stream()
            for _ in range(reps):
                start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                start.record(stream)
                run_kernel_async(kernel, graph, dev, extents, outs, stream)
                stop.record(stream)
                stop.synchronize()
                best = min(best, start.elapsed_time(stop) * 1e-3)
        except Exception as exc:
            return failure("runtime-crash", repr(exc))
        return CostReport(total=best, source="empirical")
    finally:
        try:
            _native.set_tuning(**saved)
        except Exception:
            pass


class GpuEmpiricalTimer:
    """Fitness that validates and times a variant on the current CUDA device.
    Evaluations are serialised (one launch sequence at a time on the device)."""

    parallel_safe = False

    def __init__(self, graph: TypedSpec, extents: dict | None = None, reps: int = 5,
                 validate_extents: dict | None = None, fault=None):
        self.graph = graph
        self.extents = extents or {n: 1000 for n in graph.extent_names}
        self.reps = reps
        self.validate_extents = validate_extents
        self.fault = fault
        match_corpus(graph.spec)

    def key_salt(self) -> str:
        return "empirical-gpu:" + ",".join(f"{k}={v}" for k, v in sorted(self.extents.items()))

    def __call__(self, variant: GpuVariant) -> CostReport:
        return measure_empirical(variant, self.graph, self.extents, self.reps,
                                 validate_extents=self.validate_extents, fault=self.fault)


class FitnessMemo:
    """A fitness function behind a memo table (the role of cost.py:211-237).

    The table is keyed by `<salt>|<variant key>`, the salt being whatever the wrapped
    fitness reports through `key_salt()` (extents, device), so one memo can never hand a
    timing taken at one problem size to a search at another.  `lookup()` answers from
    the table without evaluating -- the search driver uses it to decide whether a
    candidate would cost a fresh evaluation before it spends budget on it."""

    def __init__(self, fn, enabled: bool = True):
        self.fn = fn
        self.enabled = bool(enabled)
        self.parallel_safe = bool(getattr(fn, "parallel_safe", False))
        self._reports: dict[str, CostReport] = {}
        self._lookups = 0          # calls answered from the table
        self._evaluations = 0      # calls that ran the wrapped fitness

    # -- counters under the names the reference's summary.json uses -------------------
    @property
    def hits(self) -> int:
        return self._lookups

    @property
    def misses(self) -> int:
        return self._evaluations

    def key(self, variant: GpuVariant) -> str:
        salt_of = getattr(self.fn, "key_salt", None)
        return f"{salt_of() if salt_of else ''}|{variant.key()}"

    def lookup(self, variant: GpuVariant) -> CostReport | None:
        return self._reports.get(self.key(variant)) if self.enabled else None

    def __call__(self, variant: GpuVariant) -> CostReport:
        known = self.lookup(variant)
        if known is not None:
            self._lookups += 1
            return known
        self._evaluations += 1
        report = self.fn(variant)
        if self.enabled:
            self._reports[self.key(variant)] = report
        return report


CachedFitness = FitnessMemo        # the name callers of the reference's protocol know


def cached(fn, enabled: bool = True) -> FitnessMemo:
    return fn if isinstance(fn, FitnessMemo) and fn.enabled == enabled else FitnessMemo(fn, enabled)


def variant_space(kernel: str) -> list[GpuVariant]:
    """The launch variants worth timing for `kernel` (what scripts/sweep.py walks)."""
    kernel = kernel.lower()
    if kernel in ("axpydot", "vadd", "waxpby"):
        return [GpuVariant(kernel, (("vec_unroll", u), ("vec_grid_per_sm", g)))
                for u in (1, 2, 4) for g in (0, 4, 8, 16)]
    out = []
    if kernel in ("atax", "batax"):
        out += [GpuVariant(kernel, (("atax_fused", 1), ("atax_cluster", c), ("atax_rows", r)))
                for c in (0, 4, 8, 9) for r in (0, 1)]
        out.append(GpuVariant(kernel, (("atax_fused", 0),)))
        return out
    for rows, vec in ((8, 1), (16, 1), (8, 2)):
        for minb in (1, 2, 4):
            for grid in (0, 2, 8):
                out.append(GpuVariant(kernel, (("mv_rows", rows), ("mv_vec", vec),
                                               ("mv_minb", minb), ("grid_per_sm", grid))))
    return out


def tune(graph: TypedSpec, extents: dict, fitness=None, space=None) -> tuple[GpuVariant, CostReport]:
    """Exhaustive walk of the (small) variant space; returns the fastest valid variant."""
    name = match_corpus(graph.spec)
    fitness = fitness or cached(GpuEmpiricalTimer(graph, extents))
    best = None
    for variant in (space or variant_space(name)):
        report = fitness(variant)
        if not report.failed and (best is None or report.total < best[1].total):
            best = (variant, report)
    if best is None:
        raise RuntimeError(f"no variant of {name} validated")
    return best
