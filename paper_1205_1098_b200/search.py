"""Search over GPU launch variants: the GPU-side counterpart of `matfuse.search`.

The reference searches fuse-set forests (organisms) with a greedy seed plus a
genetic algorithm and writes an append-only `log.jsonl` and a `summary.json`
(`search.py:722-896`, `cli.py:219-246`).  On the GPU the fused loop structure of
every corpus kernel is fixed by the hand-written sequence, so what remains to be
searched is the launch geometry: the `GpuVariant` tunables of
`include/bto_b200.h` section 4.  This module keeps the reference's driver
protocol -- `run_strategy(strategy, graph, cfg, fitness) -> SearchResult`, a
unique-evaluation budget, an incumbent, a log in the same schema -- over that
space, with strategies

    "default"     the shipped per-kind defaults only (the max-fuse seed's role)
    "exhaustive"  every variant of `cost.variant_space`
    "random"      uniform draws from the space
    "ga"          tournament selection + one-gene mutation / uniform crossover

`fitness` is any callable `GpuVariant -> CostReport` (cost.AnalyticGpuCost,
cost.GpuEmpiricalTimer, or a CachedFitness around either).
"""
from __future__ import annotations

import json
import random
import time
from dataclasses import dataclass, field
from pathlib import Path

from .cost import CostReport, GpuVariant, cached, variant_space
from .spec import match_corpus

__all__ = ["SearchConfig", "LogEntry", "SearchResult", "run_strategy", "write_run", "STRATEGIES",
           "Autotuner"]

STRATEGIES = ("default", "exhaustive", "random", "ga")


@dataclass(frozen=True)
class SearchConfig:
    """Knobs of one search run.  The field names are the reference's (`search.py:37-50`,
    they appear in its CLI and in `summary.json`); only the ones that mean something for a
    launch-variant search exist here."""
    population: int = 8
    tournament_k: int = 2
    generations: int = 10
    budget: int | None = None          # cap on fresh (not memoised) evaluations; None = no cap
    time_budget_s: float | None = None  # cap on wall-clock seconds; None = no cap
    seed: int = 0
    mutation_prob: float = 0.5

    def __post_init__(self):
        problems = []
        if self.population < 2:
            problems.append("population must be at least 2")
        if self.tournament_k < 1:
            problems.append("tournament size must be at least 1")
        if not 0.0 <= self.mutation_prob <= 1.0:
            problems.append("mutation_prob must lie in [0, 1]")
        if problems:
            raise ValueError("; ".join(problems))


#: one line of log.jsonl -- the schema is the reference's (cli.py:227-233)
LOG_FIELDS = ("key", "fitness", "generation", "elapsed_s", "strategy")


@dataclass
class LogEntry:
    key: str
    fitness: float
    generation: int
    elapsed_s: float
    strategy: str

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name in LOG_FIELDS}


@dataclass
class SearchResult:
    strategy: str
    best: GpuVariant
    best_fitness: float
    best_report: CostReport
    log: list[LogEntry] = field(default_factory=list)
    evaluations: int = 0
    cache_hits: int = 0

    @property
    def best_key(self) -> str:
        return self.best.key()


class SearchExhausted(Exception):
    """Raised by the ledger when the next candidate would exceed a budget."""


class _Ledger:
    """Book-keeping of one search run: every candidate goes through `price()`.

    A candidate the memo already knows is free.  A fresh one is charged against the
    evaluation budget and the time budget BEFORE it is evaluated (so a budget of k never
    runs a k+1-th kernel); the very first evaluation -- the shipped defaults -- is exempt,
    which is the reference's rule too (a search always returns something).  Fresh
    evaluations are logged in order and the incumbent is the lexicographic minimum of
    (fitness, key), so ties do not depend on visiting order."""

    def __init__(self, fitness, strategy: str, cfg: SearchConfig):
        self.memo = cached(fitness)
        self.strategy, self.cfg = strategy, cfg
        self.generation = 0
        self.entries: list[LogEntry] = []
        self.incumbent: GpuVariant | None = None
        self.incumbent_report: CostReport | None = None
        self._started = time.perf_counter()
        self._charged = 0

    def _elapsed(self) -> float:
        return time.perf_counter() - self._started

    def _afford(self) -> None:
        if self._charged == 0:
            return
        if self.cfg.budget is not None and self._charged >= self.cfg.budget:
            raise SearchExhausted("evaluation budget")
        if self.cfg.time_budget_s is not None and self._elapsed() > self.cfg.time_budget_s:
            raise SearchExhausted("time budget")

    def price(self, variant: GpuVariant) -> float:
        report = self.memo.lookup(variant)
        if report is None:
            self._afford()
            report = self.memo(variant)
            self._charged += 1
            # an analytic model has no meaningful clock: keep its logs reproducible
            stamp = 0.0 if report.source == "analytic" else self._elapsed()
            self.entries.append(LogEntry(variant.key(), report.total, self.generation, stamp,
                                         self.strategy))
            if self.incumbent is None or \
                    (report.total, variant.key()) < (self.incumbent_report.total, self.incumbent.key()):
                self.incumbent, self.incumbent_report = variant, report
        else:
            self.memo(variant)                 # counted as a cache hit
        return report.total

    def result(self) -> SearchResult:
        if self.incumbent is None:
            raise RuntimeError("the search evaluated nothing")
        return SearchResult(self.strategy, self.incumbent, self.incumbent_report.total,
                            self.incumbent_report, self.entries, self.memo.misses, self.memo.hits)


def _gene_pool(space: list[GpuVariant]) -> dict[str, list[int]]:
    pool: dict[str, set[int]] = {}
    for v in space:
        for k, val in v.tuning:
            pool.setdefault(k, set()).add(val)
    return {k: sorted(vals) for k, vals in pool.items()}


def _mutate(v: GpuVariant, pool: dict[str, list[int]], rng: random.Random) -> GpuVariant:
    genes = dict(v.tuning)
    candidates = [k for k in genes if len(pool.get(k, ())) > 1]
    if not candidates:
        return v
    k = rng.choice(candidates)
    genes[k] = rng.choice([x for x in pool[k] if x != genes[k]])
    return GpuVariant(v.kernel, tuple(sorted(genes.items())))


def _crossover(a: GpuVariant, b: GpuVariant, rng: random.Random) -> GpuVariant:
    ga, gb = dict(a.tuning), dict(b.tuning)
    if set(ga) != set(gb):          # different shapes of variant (e.g. fused vs two-pass ATAX)
        return a if rng.random() < 0.5 else b
    child = {k: (ga[k] if rng.random() < 0.5 else gb[k]) for k in ga}
    return GpuVariant(a.kernel, tuple(sorted(child.items())))


def run_strategy(strategy: str, graph, cfg: SearchConfig, fitness,
                 space: list[GpuVariant] | None = None) -> SearchResult:
    """Search the launch variants of `graph`'s kernel; lower fitness is better."""
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}; expected one of {STRATEGIES}")
    kernel = match_corpus(graph.spec)
    space = list(space) if space is not None else variant_space(kernel)
    space = [GpuVariant(v.kernel, tuple(sorted(v.tuning))) for v in space]
    rng = random.Random(cfg.seed)
    ledger = _Ledger(fitness, strategy, cfg)
    try:
        ledger.price(GpuVariant(kernel))         # the shipped defaults are always evaluated
        if strategy == "exhaustive":
            for v in space:
                ledger.price(v)
        elif strategy == "random":
            draws = cfg.budget if cfg.budget is not None else cfg.population * cfg.generations
            for _ in range(draws):
                ledger.price(rng.choice(space))
        elif strategy == "ga":
            _evolve(ledger, space, cfg, rng)
    except SearchExhausted:
        pass
    return ledger.result()


def _evolve(ledger: _Ledger, space: list[GpuVariant], cfg: SearchConfig, rng: random.Random) -> None:
    """Generational GA over launch variants: k-tournament parents, uniform crossover,
    one-gene mutation, and the incumbent re-inserted whenever a generation lost it."""
    pool = _gene_pool(space)

    def scored(v: GpuVariant):
        return v, ledger.price(v)

    def tournament(population):
        entrants = rng.sample(population, min(cfg.tournament_k, len(population)))
        return min(entrants, key=lambda pair: pair[1])[0]

    population = [scored(rng.choice(space)) for _ in range(cfg.population)]
    for generation in range(1, cfg.generations + 1):
        ledger.generation = generation
        offspring = []
        for _ in range(cfg.population):
            child = _crossover(tournament(population), tournament(population), rng)
            if rng.random() < cfg.mutation_prob:
                child = _mutate(child, pool, rng)
            offspring.append(scored(child))
        champion, champion_fit = ledger.incumbent, ledger.incumbent_report.total
        if all(fit > champion_fit for _, fit in offspring):
            loser = max(range(len(offspring)), key=lambda i: (offspring[i][1], offspring[i][0].key()))
            offspring[loser] = (champion, champion_fit)
        population = offspring


def write_run(outdir, graph, result: SearchResult, cfg: SearchConfig, fitness_source: str) -> dict:
    """`log.jsonl` (append-only) and `summary.json`, the reference's formats
    (cli.py:227-246); returns the summary."""
    outdir = Path(outdir)
    outdir.mkdir(parents=True, exist_ok=True)
    with (outdir / "log.jsonl").open("a") as fh:
        for entry in result.log:
            fh.write(json.dumps(entry.as_dict()) + "\n")
    summary = {
        "kernel": graph.spec.name,
        "strategy": result.strategy,
        "best": result.best_key,
        "fitness": result.best_fitness,
        "evaluations": result.evaluations,
        "cache_hits": result.cache_hits,
        "seed": cfg.seed,
        "fitness_source": fitness_source,
    }
    (outdir / "summary.json").write_text(json.dumps(summary, indent=2) + "\n")
    return summary


# ---------------------------------------------------------------------------
# persistent tuning: search once per (kernel, extents), reuse afterwards

class Autotuner:
    """BTO's thesis -- pick the variant by measuring -- as a cache in front of the
    library: `best(graph, extents)` searches the launch variants once (empirical
    fitness by default), stores the winner in a JSON file keyed by kernel, extents and
    device, and returns it from the file afterwards; `applied(variant)` is a context
    manager that installs the variant's tunables for the duration of a call and
    restores the previous ones."""

    def __init__(self, path, strategy: str = "exhaustive", cfg: SearchConfig | None = None,
                 fitness_factory=None, device_tag: str | None = None):
        self.path = Path(path)
        self.strategy, self.cfg = strategy, cfg or SearchConfig()
        self.fitness_factory = fitness_factory
        self.device_tag = device_tag
        self._table = json.loads(self.path.read_text()) if self.path.exists() else {}

    def _key(self, kernel: str, extents: dict) -> str:
        if self.device_tag is None:
            try:
                from ._native import device_info
                info = device_info()
                self.device_tag = f"sm{info['sm_count']}"
            except Exception:           # no device: analytic tuning only
                self.device_tag = "nodevice"
        ext = ",".join(f"{k}={int(v)}" for k, v in sorted(extents.items()))
        return f"{kernel}|{ext}|{self.device_tag}"

    def best(self, graph, extents: dict) -> GpuVariant:
        kernel = match_corpus(graph.spec)
        key = self._key(kernel, extents)
        if key in self._table:
            entry = self._table[key]
            return GpuVariant(kernel, tuple((k, int(v)) for k, v in entry["tuning"]))
        if self.fitness_factory is not None:
            fitness = self.fitness_factory(graph, extents)
        else:
            from .cost import GpuEmpiricalTimer
            fitness = cached(GpuEmpiricalTimer(graph, extents))
        result = run_strategy(self.strategy, graph, self.cfg, fitness)
        self._table[key] = {"tuning": [list(kv) for kv in result.best.tuning],
                            "fitness": result.best_fitness, "strategy": self.strategy,
                            "evaluations": result.evaluations}
        self.path.parent.mkdir(parents=True, exist_ok=True)
        self.path.write_text(json.dumps(self._table, indent=1, sort_keys=True) + "\n")
        return result.best

    @staticmethod
    def applied(variant: GpuVariant):
        from contextlib import contextmanager

        from . import _native

        @contextmanager
        def scope():
            saved = {k: _native.get_tuning(k) for k, _ in variant.tuning}
            _native.set_tuning(**dict(variant.tuning))
            try:
                yield variant
            finally:
                _native.set_tuning(**saved)

        return scope()


# ---------------------------------------------------------------------------
# command line: the `--fitness` entry of the reference's `matfuse search` (cli.py:205-246)
# for the GPU cost model and the GPU timer.  Same exit codes (cli.py:42-44), same output files.

EXIT_USAGE, EXIT_KERNEL, EXIT_TOOLCHAIN = 1, 2, 3


def main(argv=None) -> int:
    """python -m paper_1205_1098_b200 search KERNEL [--strategy ga] [--fitness analytic|gpu]
    [--extents M=4096,N=4096] [--out-dir DIR] [--budget K] [--seed S] [--reps R]

    KERNEL is a corpus kernel name or the path of a `.bto` file with a corpus structure.
    `--fitness analytic` prices launch variants with the HBM-bytes / occupancy model (no GPU
    needed), `--fitness gpu` validates and times them on the current CUDA device."""
    import argparse
    import sys

    from .cost import AnalyticGpuCost, GpuEmpiricalTimer, GpuMachineModel
    from .runtime import load_graph
    from .spec import infer_shapes, parse_kernel

    ap = argparse.ArgumentParser(prog="python -m paper_1205_1098_b200 search", description=main.__doc__)
    ap.add_argument("kernel")
    ap.add_argument("--strategy", choices=STRATEGIES, default="ga")
    ap.add_argument("--fitness", choices=("analytic", "gpu"), default="analytic")
    ap.add_argument("--extents", default="M=4096,N=4096")
    ap.add_argument("--out-dir", default="search-out")
    ap.add_argument("--budget", type=int, default=None)
    ap.add_argument("--time-budget", type=float, default=None)
    ap.add_argument("--population", type=int, default=8)
    ap.add_argument("--generations", type=int, default=10)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    try:
        args = ap.parse_args(argv)
    except SystemExit as exc:
        return EXIT_USAGE if exc.code else 0
    try:
        extents = {k: int(v) for k, v in (kv.split("=") for kv in args.extents.split(","))}
        path = Path(args.kernel)
        graph = infer_shapes(parse_kernel(path.read_text())) if path.suffix == ".bto" and path.exists() \
            else load_graph(args.kernel)
        match_corpus(graph.spec)
        cfg = SearchConfig(population=args.population, generations=args.generations, budget=args.budget,
                           time_budget_s=args.time_budget, seed=args.seed)
    except (ValueError, KeyError, OSError, NotImplementedError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    if args.fitness == "gpu":
        try:
            import torch
            from . import _native
            _native.load()
            if not torch.cuda.is_available():
                raise RuntimeError("no CUDA device")
        except Exception as exc:
            print(f"error: the gpu fitness needs libbto_b200.so and a B200 ({exc})", file=sys.stderr)
            return EXIT_TOOLCHAIN
        fitness = cached(GpuEmpiricalTimer(graph, extents, reps=args.reps))
    else:
        fitness = cached(AnalyticGpuCost(graph, GpuMachineModel(extents=tuple(sorted(extents.items())))))
    result = run_strategy(args.strategy, graph, cfg, fitness)
    summary = write_run(args.out_dir, graph, result, cfg, args.fitness)
    print(json.dumps(summary, indent=2))
    return EXIT_KERNEL if result.best_report.failed else 0

