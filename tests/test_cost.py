"""GPU cost model (HBM bytes + occupancy) and the fitness plug-in protocol.
Mirrors the reference's tests/test_cost.py: hand counts, caching, and (on a
GPU) the empirical failure paths through fault injection."""
from __future__ import annotations

import math

import pytest

import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import cost as C

N = 32768
MACHINE = C.GpuMachineModel(extents=(("M", N), ("N", N)))


class TestTraffic:
    def test_algorithmic_bytes_match_survey_table(self):
        assert C.hbm_traffic("bicgk", N, N).algorithmic == 8 * N * N + 32 * N
        assert C.hbm_traffic("gemver", N, N).algorithmic == 24 * N * N + 72 * N
        assert C.hbm_traffic("axpydot", 1 << 27, 1).algorithmic == 32 * (1 << 27)

    def test_bicgk_partials_hand_count(self):
        # defaults: 8-row units, 512-column strips -> 64 strips; q partials are
        # nstrips*M doubles written + read; s partials slots*N doubles likewise
        t = C.hbm_traffic("bicgk", N, N)
        nstrips, grid = 64, 148 * 8
        slots = -(-grid // nstrips) + 1
        assert t.partials == 2 * 8 * nstrips * N + 2 * 8 * slots * N
        assert t.partials < 0.01 * t.algorithmic
        assert t.rereads == 0 and t.launches == 2

    def test_two_pass_atax_rereads_the_matrix(self):
        fused = C.hbm_traffic("atax", N, N, C.GpuVariant("atax", (("atax_fused", 1),)))
        split = C.hbm_traffic("atax", N, N, C.GpuVariant("atax", (("atax_fused", 0),)))
        assert fused.rereads == 0
        assert split.rereads == 8 * N * N
        assert split.launches == 4 and fused.launches == 2

    def test_gemver_counts_the_write_and_reread_of_B(self):
        # the reference's distinct-array rule counts B once (cost.py:80-86)
        t = C.hbm_traffic("gemver", N, N)
        kinds = [p[0] for p in t.passes]
        assert kinds == ["TR", "N"]
        assert t.passes[0][1] == 8 * N * N and t.passes[0][2] == 8 * N * N
        assert t.passes[1][1] == 8 * N * N


def test_atax_cluster_choice_restates_the_library_plan():
    """cost.atax_cluster_choice is the Python restatement of plan_atax (host_sequences.cuh); the GPU
    test test_atax_cluster_size_follows_the_slice_width holds the library to the same picks."""
    picks = {n: C.atax_cluster_choice(n)[:3] for n in (8192, 12288, 20480, 24576, 32768, 40960, 2048, 20000)}
    assert picks[8192] == (2, 8, 2) and picks[12288] == (3, 8, 2) and picks[20480] == (5, 8, 2)
    assert picks[24576] == (6, 8, 2) and picks[32768] == (9, 8, 2) and picks[40960] == (10, 8, 2)
    assert picks[2048][0] == 1 and picks[20000][0] in (5, 9)
    with pytest.raises(ValueError):
        C.atax_cluster_choice(16 * 8192 + 2)


class TestAnalytic:
    def test_fused_atax_beats_two_pass(self):
        g = bto.load_graph("atax")
        fused = C.estimate_cost(C.GpuVariant("atax", (("atax_fused", 1),)), g, MACHINE)
        split = C.estimate_cost(C.GpuVariant("atax", (("atax_fused", 0),)), g, MACHINE)
        assert fused.total < 0.6 * split.total
        assert fused.contracted == ("t0",)

    def test_estimates_land_near_measured_times(self):
        # profiles/r01: bicgk 1.21 ms, gesummv 1.37 ms, gemver 3.97 ms at bench sizes
        for name, ext, ms in (("bicgk", (N, N), 1.21), ("gemver", (N, N), 3.97),
                              ("gesummv", (24576, 24576), 1.37)):
            m = C.GpuMachineModel(extents=(("M", ext[0]), ("N", ext[1])))
            est = C.estimate_cost(C.GpuVariant(name), bto.load_graph(name), m).total * 1e3
            assert abs(est - ms) / ms < 0.15, (name, est)

    def test_starved_grid_is_latency_bound(self):
        g = bto.load_graph("bicgk")
        full = C.estimate_cost(C.GpuVariant("bicgk"), g, MACHINE).total
        starved = C.estimate_cost(C.GpuVariant("bicgk", (("grid_per_sm", 1), ("mv_minb", 1))),
                                  g, MACHINE).total
        assert starved > 1.5 * full

    def test_pure_function_and_breakdown(self):
        g = bto.load_graph("gemver")
        a = C.estimate_cost(C.GpuVariant("gemver"), g, MACHINE)
        b = C.estimate_cost(C.GpuVariant("gemver"), g, MACHINE)
        assert a == b
        assert math.isclose(sum(a.per_root), a.total)
        assert a.partition_nodes == 4 and a.source == "analytic" and not a.failed

    def test_sharded_variants_pay_one_collective(self):
        g = bto.load_graph("bicgk")
        one = C.estimate_cost(C.GpuVariant("bicgk"), g, MACHINE).total
        eight = C.estimate_cost(C.GpuVariant("bicgk", (("world", 8),)), g, MACHINE).total
        assert math.isclose(eight - one, MACHINE.collective_us * 1e-6)
        g2 = bto.load_graph("gesummv")       # y stays sharded: no exchange
        assert C.estimate_cost(C.GpuVariant("gesummv", (("world", 8),)), g2, MACHINE).total == \
            C.estimate_cost(C.GpuVariant("gesummv"), g2, MACHINE).total


class TestCaching:
    class Counting:
        parallel_safe = True

        def __init__(self):
            self.calls = 0

        def key_salt(self):
            return "count"

        def __call__(self, variant):
            self.calls += 1
            return C.estimate_cost(variant, None, MACHINE)

    def test_same_variant_evaluates_once(self):
        fn = C.cached(self.Counting())
        v = C.GpuVariant("bicgk", (("mv_rows", 8),))
        fn(v)
        fn(C.GpuVariant("bicgk", (("mv_rows", 8),)))
        assert fn.fn.calls == 1 and fn.hits == 1 and fn.misses == 1

    def test_tuning_distinguishes_keys(self):
        fn = C.cached(self.Counting())
        fn(C.GpuVariant("bicgk", (("mv_rows", 8),)))
        fn(C.GpuVariant("bicgk", (("mv_rows", 16),)))
        assert fn.fn.calls == 2

    def test_disabled_cache(self):
        fn = C.cached(self.Counting(), enabled=False)
        v = C.GpuVariant("bicgk")
        fn(v)
        fn(v)
        assert fn.fn.calls == 2


def test_variant_space_is_nonempty_for_every_corpus_kernel():
    for name in bto.CORPUS:
        assert C.variant_space(name), name


@pytest.mark.gpu
class TestEmpirical:
    def test_variant_validates_and_times(self):
        g = bto.load_graph("gemver")
        rep = C.measure_empirical(C.GpuVariant("gemver"), g, {"M": 2048, "N": 2048}, reps=3)
        assert rep.source == "empirical" and not rep.failed and 0 < rep.total < 1e-2

    def test_wrong_answers_never_get_finite_fitness(self):
        g = bto.load_graph("bicgk")

        def corrupt(outs):
            outs = dict(outs)
            outs["s"] = outs["s"] * (1 + 1e-6)
            return outs

        rep = C.measure_empirical(C.GpuVariant("bicgk"), g, {"M": 512, "N": 512}, reps=1,
                                  fault=corrupt)
        assert rep.failed and rep.diagnostic.startswith("numerical-mismatch")

    def test_unsupported_tuning_reports_compile_failure(self):
        g = bto.load_graph("bicgk")
        rep = C.measure_empirical(C.GpuVariant("bicgk", (("mv_rows", 5),)), g,
                                  {"M": 512, "N": 512}, reps=1)
        assert rep.failed and rep.diagnostic.startswith("compile-failure")

    def test_timer_class_and_tune(self):
        g = bto.load_graph("atax")
        timer = C.cached(C.GpuEmpiricalTimer(g, {"M": 4096, "N": 4096}, reps=2))
        space = [C.GpuVariant("atax", (("atax_fused", f),)) for f in (0, 1)]
        best, rep = C.tune(g, {"M": 4096, "N": 4096}, fitness=timer, space=space)
        assert not rep.failed and best in space
        assert timer.misses == 2


def test_max_rel_error_is_loud_about_unwritten_outputs():
    """Outputs arrive NaN-prefilled so that an unwritten element is visible (runtime.py:108,130);
    the reference's metric swallows the NaN (`max(0.0, nan)` is 0.0) -- ours must not."""
    import math
    import numpy as np
    want = {"y": np.ones(4), "beta": 2.0}
    assert bto.max_rel_error({"y": np.ones(4), "beta": 2.0}, want) == 0.0
    assert bto.max_rel_error({"y": np.array([1.0, np.nan, 1.0, 1.0]), "beta": 2.0}, want) == math.inf
    assert bto.max_rel_error({"y": np.ones(4), "beta": float("nan")}, want) == math.inf
    assert bto.max_rel_error({"y": np.array([1.0, np.inf, 1.0, 1.0]), "beta": 2.0}, want) == math.inf
    assert bto.max_rel_error({"y": np.ones(3), "beta": 2.0}, want) == math.inf       # wrong length


def test_validation_extents_keep_the_timed_dispatch():
    """Validation runs at the timed extents, or at the same N with fewer rows when the in-product
    evaluator's temporaries would not fit -- never at min(64, extent)."""
    assert C.validation_extents({"M": 4096, "N": 4096}) == {"M": 4096, "N": 4096}
    assert C.validation_extents({"M": 1 << 27}) == {"M": 1 << 27}
    big = C.validation_extents({"M": 32768, "N": 32768})
    assert big["N"] == 32768 and 4096 <= big["M"] < 32768
    assert C.validation_extents({"M": 8, "N": 1 << 24}) == {"M": 8, "N": 1 << 24}
