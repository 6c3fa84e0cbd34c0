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

from .cost import CachedFitness, CostReport, GpuVariant, cached, variant_space
from .spec import match_corpus

__all__ = ["SearchConfig", "LogEntry", "SearchResult", "run_strategy", "write_run", "STRATEGIES",
           "Autotuner"]

STRATEGIES = ("default", "exhaustive", "random", "ga")


@dataclass(frozen=True)
class SearchConfig:
    population: int = 8
    tournament_k: int = 2
    generations: int = 10
    budget: int | None = None          # max unique (cache-miss) evaluations
    time_budget_s: float | None = None
    seed: int = 0
    mutation_prob: float = 0.5

    def __post_init__(self):
        if self.population < 2:
            raise ValueError("population must be at least 2")
        if self.tournament_k < 1:
            raise ValueError("tournament size must be at least 1")


@dataclass
class LogEntry:
    key: str
    fitness: float
    generation: int
    elapsed_s: float
    strategy: str

    def as_dict(self) -> dict:
        return {"key": self.key, "fitness": self.fitness, "generation": self.generation,
                "elapsed_s": self.elapsed_s, "strategy": self.strategy}


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


class _BudgetDone(Exception):
    pass


class _Evaluator:
    """Cached fitness with logging, an incumbent and a unique-evaluation budget
    (same rules as the reference's: the seed evaluation is always allowed)."""

    def __init__(self, fitness, strategy: str, cfg: SearchConfig):
        self.fitness = fitness if isinstance(fitness, CachedFitness) else cached(fitness)
        self.strategy, self.cfg = strategy, cfg
        self.log: list[LogEntry] = []
        self.generation = 0
        self.best: tuple[float, str, GpuVariant] | None = None
        self.best_report: CostReport | None = None
        self.t0 = time.perf_counter()

    def __call__(self, variant: GpuVariant) -> CostReport:
        key = self.fitness.key(variant)
        fresh = key not in self.fitness._table
        if fresh:
            if self.cfg.budget is not None and self.fitness.misses > 0 \
                    and self.fitness.misses >= self.cfg.budget:
                raise _BudgetDone()
            if self.cfg.time_budget_s is not None \
                    and time.perf_counter() - self.t0 > self.cfg.time_budget_s:
                raise _BudgetDone()
        report = self.fitness(variant)
        if fresh:
            elapsed = 0.0 if report.source == "analytic" else time.perf_counter() - self.t0
            self.log.append(LogEntry(variant.key(), report.total, self.generation, elapsed,
                                     self.strategy))
            ranked = (report.total, variant.key())
            if self.best is None or ranked < self.best[:2]:
                self.best = (report.total, variant.key(), variant)
                self.best_report = report
        return report

    def result(self) -> SearchResult:
        assert self.best is not None, "no evaluations happened"
        return SearchResult(self.strategy, self.best[2], self.best[0], self.best_report, self.log,
                            self.fitness.misses, self.fitness.hits)


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
    seed_variant = GpuVariant(kernel)
    rng = random.Random(cfg.seed)
    ev = _Evaluator(fitness, strategy, cfg)
    try:
        ev(seed_variant)                         # the shipped defaults are always evaluated
        if strategy == "exhaustive":
            for v in space:
                ev(v)
        elif strategy == "random":
            draws = cfg.budget if cfg.budget is not None else cfg.population * cfg.generations
            for _ in range(draws):
                ev(rng.choice(space))
        elif strategy == "ga":
            pool = _gene_pool(space)
            population = []
            for _ in range(cfg.population):
                v = rng.choice(space)
                population.append((v, ev(v).total))
            for gen in range(1, cfg.generations + 1):
                ev.generation = gen
                children = []
                for _ in range(cfg.population):
                    pa = min(rng.sample(population, min(cfg.tournament_k, len(population))),
                             key=lambda t: t[1])[0]
                    pb = min(rng.sample(population, min(cfg.tournament_k, len(population))),
                             key=lambda t: t[1])[0]
                    child = _crossover(pa, pb, rng)
                    if rng.random() < cfg.mutation_prob:
                        child = _mutate(child, pool, rng)
                    children.append((child, ev(child).total))
                # elitism: the incumbent survives every generation
                best_fit, _, best_variant = ev.best
                if min(s for _, s in children) > best_fit:
                    worst = max(range(len(children)), key=lambda i: (children[i][1], children[i][0].key()))
                    children[worst] = (best_variant, best_fit)
                population = children
    except _BudgetDone:
        pass
    return ev.result()


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
