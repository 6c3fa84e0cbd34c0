"""Variant search driver: budgets, determinism, incumbent, log/summary formats.
Hermetic: the analytic cost model is the fitness (as in the reference's
tests/test_search.py); one GPU test runs the empirical timer through it."""
from __future__ import annotations

import json

import pytest

import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cost as C
from paper_1205_1098_b200 import search as S

MACHINE = C.GpuMachineModel(extents=(("M", 32768), ("N", 32768)))


def fitness(name):
    return C.cached(C.AnalyticGpuCost(bto.load_graph(name), MACHINE))


@pytest.mark.parametrize("strategy", S.STRATEGIES)
def test_every_strategy_returns_a_valid_incumbent(strategy):
    g = bto.load_graph("bicgk")
    res = S.run_strategy(strategy, g, S.SearchConfig(seed=1), fitness("bicgk"))
    assert res.best.kernel == "bicgk" and not res.best_report.failed
    assert res.best_fitness == min(e.fitness for e in res.log)
    assert res.evaluations == len(res.log) >= 1
    assert res.log[0].key == "bicgk{}"                 # the shipped defaults come first


def test_exhaustive_visits_the_whole_space_and_finds_the_minimum():
    g = bto.load_graph("atax")
    fn = fitness("atax")
    res = S.run_strategy("exhaustive", g, S.SearchConfig(), fn)
    space = C.variant_space("atax")
    assert res.evaluations == len({v.key() for v in space} | {"atax{}"})
    assert res.best_fitness == min(fn(v).total for v in space + [C.GpuVariant("atax")])
    assert res.best.get("atax_fused", 1) == 1          # single pass beats two passes


def test_budget_caps_unique_evaluations():
    g = bto.load_graph("gemver")
    res = S.run_strategy("ga", g, S.SearchConfig(budget=5, seed=3), fitness("gemver"))
    assert res.evaluations <= 5
    res0 = S.run_strategy("exhaustive", g, S.SearchConfig(budget=0), fitness("gemver"))
    assert res0.evaluations == 1                        # the seed is always allowed


def test_search_is_deterministic_for_a_seed():
    g = bto.load_graph("gesummv")
    a = S.run_strategy("ga", g, S.SearchConfig(seed=7, generations=4), fitness("gesummv"))
    b = S.run_strategy("ga", g, S.SearchConfig(seed=7, generations=4), fitness("gesummv"))
    assert [e.key for e in a.log] == [e.key for e in b.log] and a.best_key == b.best_key


def test_ga_never_loses_the_incumbent():
    g = bto.load_graph("bicgk")
    res = S.run_strategy("ga", g, S.SearchConfig(seed=2, generations=6), fitness("bicgk"))
    best_so_far = float("inf")
    for e in res.log:
        best_so_far = min(best_so_far, e.fitness)
    assert res.best_fitness == best_so_far


def test_log_and_summary_formats(tmp_path):
    g = bto.load_graph("bicgk")
    cfg = S.SearchConfig(seed=5)
    res = S.run_strategy("random", g, cfg, fitness("bicgk"))
    summary = S.write_run(tmp_path, g, res, cfg, "analytic")
    lines = [json.loads(l) for l in (tmp_path / "log.jsonl").read_text().splitlines()]
    assert len(lines) == len(res.log)
    assert set(lines[0]) == {"key", "fitness", "generation", "elapsed_s", "strategy"}
    assert json.loads((tmp_path / "summary.json").read_text()) == summary
    assert set(summary) == {"kernel", "strategy", "best", "fitness", "evaluations", "cache_hits",
                            "seed", "fitness_source"}
    S.write_run(tmp_path, g, res, cfg, "analytic")       # append-only log
    assert len((tmp_path / "log.jsonl").read_text().splitlines()) == 2 * len(res.log)


def test_unknown_strategy_and_unsupported_kernel():
    g = bto.load_graph("bicgk")
    with pytest.raises(ValueError):
        S.run_strategy("annealing", g, S.SearchConfig(), fitness("bicgk"))


@pytest.mark.gpu
def test_empirical_search_on_device():
    g = bto.load_graph("bicgk")
    timer = C.cached(C.GpuEmpiricalTimer(g, {"M": 4096, "N": 4096}, reps=2))
    space = [C.GpuVariant("bicgk", (("mv_minb", b), ("mv_rows", 8))) for b in (1, 4)]
    res = S.run_strategy("exhaustive", g, S.SearchConfig(), timer, space=space)
    assert res.evaluations == 3 and not res.best_report.failed
    assert all(e.elapsed_s > 0 for e in res.log)


def test_autotuner_searches_once_and_persists(tmp_path):
    calls = []

    def factory(graph, extents):
        calls.append(dict(extents))
        m = C.GpuMachineModel(extents=tuple(sorted(extents.items())))
        return C.cached(C.AnalyticGpuCost(graph, m))

    g = bto.load_graph("atax")
    path = tmp_path / "cache" / "tuned.json"
    tuner = S.Autotuner(path, fitness_factory=factory, device_tag="test")
    a = tuner.best(g, {"M": 4096, "N": 4096})
    b = tuner.best(g, {"M": 4096, "N": 4096})
    assert a == b and len(calls) == 1                     # second lookup is served from the table
    tuner.best(g, {"M": 8192, "N": 4096})
    assert len(calls) == 2                                 # another shape is another search
    again = S.Autotuner(path, fitness_factory=factory, device_tag="test")
    assert again.best(g, {"M": 4096, "N": 4096}) == a and len(calls) == 2     # persisted
    table = json.loads(path.read_text())
    assert set(table) == {"atax|M=4096,N=4096|test", "atax|M=8192,N=4096|test"}
    assert set(next(iter(table.values()))) == {"tuning", "fitness", "strategy", "evaluations"}


def test_applied_variant_is_restored():
    from paper_1205_1098_b200 import _native
    before = _native.get_tuning("mv_rows")
    with S.Autotuner.applied(C.GpuVariant("bicgk", (("mv_rows", 16),))):
        assert _native.get_tuning("mv_rows") == 16
    assert _native.get_tuning("mv_rows") == before


@pytest.mark.gpu
def test_autotuner_with_the_empirical_timer(tmp_path):
    g = bto.load_graph("gesummv")
    tuner = S.Autotuner(tmp_path / "tuned.json", strategy="random", cfg=S.SearchConfig(budget=4, seed=1))
    best = tuner.best(g, {"M": 4096, "N": 4096})
    assert best.kernel == "gesummv"
    with S.Autotuner.applied(best):
        inputs = bto.gen_inputs(g, {"M": 64, "N": 64}, seed=1)
        out = bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, inputs, {"M": 64, "N": 64})
    assert out["y"].shape == (64,)


def test_command_line_search_with_the_analytic_fitness(tmp_path, capsys):
    """`python -m paper_1205_1098_b200 search` -- the `--fitness` entry of the reference's CLI
    (cli.py:205-246): same files, same exit codes."""
    from paper_1205_1098_b200.__main__ import main
    rc = main(["search", "gemver", "--strategy", "random", "--fitness", "analytic", "--extents",
               "M=8192,N=8192", "--budget", "6", "--out-dir", str(tmp_path)])
    assert rc == 0
    summary = json.loads((tmp_path / "summary.json").read_text())
    assert summary["kernel"] == "GEMVER" and summary["fitness_source"] == "analytic"
    assert 1 <= summary["evaluations"] <= 6
    assert len((tmp_path / "log.jsonl").read_text().splitlines()) == summary["evaluations"]
    assert main(["search", "no-such-kernel"]) == S.EXIT_USAGE
    assert main(["enumerate"]) == S.EXIT_USAGE
    import torch
    if not torch.cuda.is_available():
        assert main(["search", "bicgk", "--fitness", "gpu", "--out-dir", str(tmp_path)]) == S.EXIT_TOOLCHAIN
