"""Parity of the sm_100a kernels with the reference, through the C ABI.

Every test here needs a B200 (`-m gpu`).  The checker is the CPU oracle
(oracle/, bit-identical to the reference's generated C -- tests/test_oracle.py)
and the committed golden outputs of the reference itself.  Gate (BASELINE.json
north_star): max relative error <= 1e-12 * log2(n) with the reference's metric
|g - e| / max(|e|, 1) (runtime.py:167-175); outputs that involve no reduction
(AXPYDOT z, GEMVER B, VADD x, WAXPBY w) must be BIT-IDENTICAL.
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import golden_util as G
import paper_1205_1098_b200 as bto
from paper_1205_1098_b200 import _native

pytestmark = pytest.mark.gpu

KERNELS = tuple(bto.CORPUS)
ELEMENTWISE = {"axpydot": ("z",), "gemver": ("B",), "vadd": ("x",), "waxpby": ("w",)}


def tol(ext: dict) -> float:
    return 1e-12 * max(1.0, math.log2(max(ext.values())))


def ext_of(name: str, m: int, n: int) -> dict:
    return {"M": m} if bto.load_graph(name).extent_names == ("M",) else {"M": m, "N": n}


def run_host(name, inputs, ext):
    g = bto.load_graph(name)
    return bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, inputs, ext)


def run_device(name, inputs, ext):
    g = bto.load_graph(name)
    dev = {k: (torch.from_numpy(np.ascontiguousarray(v)).cuda() if isinstance(v, np.ndarray) else v)
           for k, v in inputs.items()}
    out = bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, dev, ext)
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}


def assert_matches(name, got, want, ext, what=""):
    for out in want:
        assert not np.any(np.isnan(np.asarray(got[out]))), f"{name}.{out} has unwritten (NaN) elements"
    err = bto.max_rel_error(got, want)
    assert err <= tol(ext), f"{name} {ext} {what}: error {err:.3e} > {tol(ext):.3e}"
    for out in ELEMENTWISE.get(name, ()):
        assert np.array_equal(np.asarray(got[out]), np.asarray(want[out])), \
            f"{name}.{out} {ext} {what}: not bit-identical"


@pytest.mark.parametrize("name", KERNELS)
def test_golden_small_cases_host_and_device_pointers(bto_lib, name):
    graph = bto.load_graph(name)
    for (m, n, seed) in G.small_cases(name):
        ext = ext_of(name, m, n)
        inputs = bto.random_inputs(graph, ext, seed=seed)
        prefix = f"small/{m}x{n}/s{seed}"
        for runner in (run_host, run_device):
            got = runner(name, inputs, ext)
            for which in ("O2", "O1"):
                want = G.expected(name, prefix, which)
                assert G.max_err(got, want) <= tol(ext), (name, ext, seed, which, runner.__name__)
            for out in ELEMENTWISE.get(name, ()):
                assert G.bit_equal(got[out], G.expected(name, prefix, "O2")[out]), (name, ext, out)


@pytest.mark.parametrize("name", bto.HOT_PATH)
def test_check_configs_against_reference_outputs(bto_lib, name):
    """BASELINE.json check sizes and seeds, against the reference's own outputs."""
    graph = bto.load_graph(name)
    ext = bto.CHECK_CONFIGS[name]
    inputs = bto.gen_inputs(graph, ext, seed=bto.SEEDS[name])
    assert G.sha([inputs[k] for k, _ in graph.spec.inputs]) == G.inputs_sha(name, "check")
    got = run_device(name, inputs, ext)
    for which in ("O2", "O1"):
        err = G.max_err(got, G.expected(name, "check", which))
        assert err <= tol(ext), f"{name} vs {which}: {err:.3e}"
    for out in ELEMENTWISE.get(name, ()):
        assert G.bit_equal(got[out], G.expected(name, "check", "O2")[out]), (name, out)


RAGGED = [(1, 1), (1, 513), (513, 1), (3, 1000), (1000, 3), (255, 511), (257, 1026),
          (1031, 2050), (64, 4096), (4100, 514), (129, 1537)]


@pytest.mark.parametrize("name", KERNELS)
def test_ragged_extents_against_live_oracle(bto_lib, oracle, name):
    """Edge tiles: extents that are not multiples of the strip width or the
    unit height, odd N (unaligned rows -> scalar-load path), single row/column."""
    graph = bto.load_graph(name)
    for (m, n) in RAGGED:
        ext = ext_of(name, m, n)
        inputs = bto.gen_inputs(graph, ext, seed=m * 7 + n)
        want = oracle.oracle_run(name, inputs, ext, threads=8)
        assert_matches(name, run_device(name, inputs, ext), want, ext, "device")
    ext = ext_of(name, 300, 77)
    inputs = bto.gen_inputs(graph, ext, seed=1)
    assert_matches(name, run_host(name, inputs, ext),
                   oracle.oracle_run(name, inputs, ext, threads=8), ext, "host")


@pytest.mark.parametrize("rows,vec", [(8, 1), (16, 1), (8, 2)])
def test_every_tile_variant(bto_lib, oracle, rows, vec):
    old = (_native.get_tuning("mv_rows"), _native.get_tuning("mv_vec"))
    try:
        _native.set_tuning(mv_rows=rows, mv_vec=vec)
        for name in ("bicgk", "atax", "gesummv", "gemver", "dgemv", "dgemvt", "batax"):
            graph = bto.load_graph(name)
            for (m, n) in [(777, 1300), (2048, 1024), (1500, 3000)]:
                ext = {"M": m, "N": n}
                inputs = bto.gen_inputs(graph, ext, seed=m + n)
                want = oracle.oracle_run(name, inputs, ext, threads=8)
                assert_matches(name, run_device(name, inputs, ext), want, ext, f"R{rows}V{vec}")
    finally:
        _native.set_tuning(mv_rows=old[0], mv_vec=old[1])


ATAX_SHAPES = [(2048, 1024), (8, 2), (1, 4096), (100, 514), (333, 8192), (64, 16390),
               (1000, 4098), (37, 32768), (5000, 1026), (257, 3586), (129, 28672), (75, 30000),
               (50, 24576), (40, 12288), (33, 20480), (65, 1536), (70, 2600), (21, 40960), (19, 36000)]


@pytest.mark.parametrize("cluster", [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 16])
def test_fused_atax_every_cluster_size(bto_lib, oracle, cluster):
    """Single-pass ATAX/BATAX (cluster-resident row panels, TMA ring, st.async
    exchange): every cluster size, ring depth and panel height must
    give the oracle's result; shapes include slices that leave the last CTA of
    the cluster short, fewer rows than clusters, and a single row."""
    try:
        for (m, n) in ATAX_SHAPES:
            ext = {"M": m, "N": n}
            for name in ("atax", "batax"):
                graph = bto.load_graph(name)
                inputs = bto.gen_inputs(graph, ext, seed=m + n)
                want = oracle.oracle_run(name, inputs, ext, threads=8)
                for stages, rows, per_sm in ((0, 0, 1), (2, 0, 1), (0, 1, 1), (4, 1, 1), (0, 0, 2), (2, 0, 2)):
                    if per_sm == 2 and cluster == 16:
                        continue                  # two CTAs per SM: clusters up to 9
                    _native.set_tuning(atax_fused=1, atax_cluster=cluster, atax_stages=stages,
                                       atax_rows=rows, atax_per_sm=per_sm)
                    assert_matches(name, run_device(name, inputs, ext), want, ext,
                                   f"C{cluster} S{stages} R{rows} per_sm{per_sm}")
    finally:
        _native.set_tuning(atax_fused=1, atax_cluster=0, atax_stages=0, atax_rows=0, atax_per_sm=1)


def test_no_kernel_depends_on_shared_memory_it_did_not_write(bto_lib, oracle):
    """Shared memory keeps what the previous kernel left in it.  Before every call here all of it is
    filled with NaN bit patterns (`bto_debug_poison_shared_memory`); ragged shapes -- row counts
    that leave the last panel / unit / tile short, column counts that leave slices and strips
    short -- must still give the oracle's result.  (Round 2: the single-pass ATAX multiplied the
    zero tile of a missing row with an exchange partial nobody had pushed: 0 x NaN, one result in
    37 000 fuzz cases; it now pushes all rows of a panel.)"""
    shapes = [(633, 8502), (21, 8502), (5, 4098), (1, 16390), (1031, 514), (37, 2050), (7, 50), (3, 70000),
              (257, 3586), (9, 24578), (13, 1026), (1001, 33), (77, 300), (600, 5000)]
    try:
        for name in KERNELS:
            graph = bto.load_graph(name)
            for (m, n) in shapes:
                ext = {"M": m * 3 + 1} if graph.extent_names == ("M",) else {"M": m, "N": n}
                inputs = bto.gen_inputs(graph, ext, seed=m + n)
                want = oracle.oracle_run(name, inputs, ext, threads=8)
                variants = [dict()]
                if name in ("atax", "batax"):
                    variants = [dict(atax_cluster=c, atax_per_sm=p, atax_rows=r)
                                for c in (0, 1, 2, 4, 8, 9, 16) for p in (1, 2) for r in (0, 1) if not (p == 2 and (c == 16 or r == 1))]
                for tune in variants:
                    _native.set_tuning(**tune)
                    _native.poison_shared_memory()
                    _native.poison_workspace()      # ... nor on partials no producer wrote in this call
                    assert_matches(name, run_device(name, inputs, ext), want, ext, f"poisoned {tune}")
                if (m + n) % 3 == 0:          # and through the host-pointer entry points (library stream)
                    _native.poison_all()
                    assert_matches(name, run_host(name, inputs, ext), want, ext, "poisoned, host operands")
    finally:
        _native.set_tuning(atax_cluster=0, atax_per_sm=1, atax_rows=0)


def test_atax_cluster_size_follows_the_slice_width(bto_lib):
    """The plan prices every built cluster size by the per-panel chain (host_sequences.cuh::plan_atax):
    rows whose length divides into full 4096-column slices get the cluster that makes them --
    24576 = 6 x 4096, 20480 = 5 x 4096, 40960 = 10 x 4096 -- and the bench size keeps 9; results
    are checked against cuBLAS-free closed forms (a rank-1 matrix)."""
    import torch
    # (how many clusters of a size fit depends on the chip's GPCs: at 32768 both 8 and 9 are in order)
    for n, want in ((32768, ("atax_cluster_kernel<9,8,2,1>", "atax_cluster_kernel<8,8,2,1>")),
                    (24576, ("atax_cluster_kernel<6,8,2,1>",)), (20480, ("atax_cluster_kernel<5,8,2,1>",)),
                    (40960, ("atax_cluster_kernel<10,8,2,1>",)), (12288, ("atax_cluster_kernel<3,8,2,1>",)),
                    (8192, ("atax_cluster_kernel<2,8,2,1>",))):
        m = 600
        u = torch.linspace(0.5, 1.5, m, dtype=torch.float64, device="cuda")
        v = torch.linspace(-1.0, 1.0, n, dtype=torch.float64, device="cuda")
        A = torch.outer(u, v).contiguous()                         # A = u v'
        x = torch.full((n,), 0.25, dtype=torch.float64, device="cuda")
        got = bto.run_kernel(bto.library_path(), bto.gpu_kernel(bto.load_graph("atax")), bto.load_graph("atax"),
                             {"A": A, "x": x}, {"M": m, "N": n})["y"]
        plan = _native.launch_plan()
        assert plan.startswith(want), (n, plan)      # (str.startswith takes a tuple of alternatives)
        expect = v * (float(u @ u) * float(v @ x))                 # A'(A x) = v (u'u)(v'x)
        assert float((got - expect).abs().max()) <= 1e-12 * math.log2(n) * max(1.0, float(expect.abs().max())), n


def test_two_pass_atax_fallback(bto_lib, oracle):
    """Odd N (rows not 16-byte aligned) and atax_fused=0 take the two-pass path."""
    try:
        for fused, (m, n) in ((1, (301, 1001)), (0, (2048, 1024)), (0, (700, 4100))):
            _native.set_tuning(atax_fused=fused)
            ext = {"M": m, "N": n}
            graph = bto.load_graph("atax")
            inputs = bto.gen_inputs(graph, ext, seed=5)
            want = oracle.oracle_run("atax", inputs, ext, threads=8)
            assert_matches("atax", run_device("atax", inputs, ext), want, ext, f"fused={fused}")
    finally:
        _native.set_tuning(atax_fused=1)


@pytest.mark.parametrize("grid_per_sm", [1, 3, 16])
def test_grid_size_only_changes_reduction_order(bto_lib, oracle, grid_per_sm):
    try:
        _native.set_tuning(grid_per_sm=grid_per_sm, vec_grid_per_sm=grid_per_sm)
        for name, ext in (("bicgk", {"M": 3000, "N": 2500}), ("axpydot", {"M": 1234567}),
                          ("gemver", {"M": 1200, "N": 2200})):
            graph = bto.load_graph(name)
            inputs = bto.gen_inputs(graph, ext, seed=3)
            want = oracle.oracle_run(name, inputs, ext, threads=8)
            assert_matches(name, run_device(name, inputs, ext), want, ext, f"grid{grid_per_sm}")
    finally:
        _native.set_tuning(grid_per_sm=0, vec_grid_per_sm=0)


def test_unaligned_device_pointers(bto_lib, oracle):
    """8-byte-aligned (not 16) base pointers must take the scalar-load path."""
    m, n = 300, 258
    graph = bto.load_graph("bicgk")
    inputs = bto.gen_inputs(graph, {"M": m, "N": n}, seed=9)
    want = oracle.oracle_run("bicgk", inputs, {"M": m, "N": n}, threads=8)
    pad = torch.empty(m * n + 1, dtype=torch.float64, device="cuda")
    A = pad[1:].view(m, n)
    A.copy_(torch.from_numpy(inputs["A"]))
    assert A.data_ptr() % 16 == 8
    dev = {"A": A, "p": torch.from_numpy(inputs["p"]).cuda(), "r": torch.from_numpy(inputs["r"]).cuda()}
    got = bto.run_kernel(bto.library_path(), bto.gpu_kernel(graph), graph, dev, {"M": m, "N": n})
    assert bto.max_rel_error(got, want) <= tol({"M": m, "N": n})
    # vector kernel, odd offset
    g2 = bto.load_graph("axpydot")
    k = 100001
    inp = bto.gen_inputs(g2, {"M": k}, seed=2)
    want = oracle.oracle_run("axpydot", inp, {"M": k}, threads=8)
    buf = torch.empty(3 * k + 3, dtype=torch.float64, device="cuda")
    dev = {"alpha": inp["alpha"]}
    for idx, nm in enumerate(("w", "v", "u")):
        view = buf[idx * (k + 1) + 1: idx * (k + 1) + 1 + k]
        view.copy_(torch.from_numpy(inp[nm]))
        dev[nm] = view
    got = bto.run_kernel(bto.library_path(), bto.gpu_kernel(g2), g2, dev, {"M": k})
    assert np.array_equal(got["z"].cpu().numpy(), want["z"])
    assert bto.max_rel_error(got, want) <= tol({"M": k})


def test_results_are_bit_stable_run_to_run(bto_lib):
    for name in ("axpydot", "bicgk", "gemver"):
        graph = bto.load_graph(name)
        ext = ext_of(name, 4096, 3072) if name != "axpydot" else {"M": 1 << 22}
        inputs = bto.gen_inputs(graph, ext, seed=0)
        a = run_device(name, inputs, ext)
        b = run_device(name, inputs, ext)
        for out in a:
            assert np.array_equal(np.asarray(a[out]), np.asarray(b[out])), (name, out)


def test_bad_extents_are_errors(bto_lib):
    lib = _native.load()
    x = torch.zeros(8, dtype=torch.float64, device="cuda")
    rc = lib.bto_vadd_async(x.data_ptr(), x.data_ptr(), x.data_ptr(), x.data_ptr(), 0, None)
    assert rc == 2 and lib.bto_last_error() == 2
    with pytest.raises(_native.BtoError):
        _native.check(rc)


def test_host_operand_pipeline(bto_lib, oracle):
    """Host buffers above the streaming threshold go through the panel pipeline
    (copy-in / compute / copy-out on three streams): GEMVER and AXPYDOT, many
    small panels, pageable and pinned memory, odd lengths, more panels than rows."""
    try:
        for panel_mib, (m, n) in ((1, (2100, 2050)), (8, (2048, 2048)), (1, (3, 1500000))):
            _native.set_tuning(host_pipeline=1, host_panel_mib=panel_mib)
            ext = {"M": m, "N": n}
            g = bto.load_graph("gemver")
            inputs = bto.gen_inputs(g, ext, seed=m)
            want = oracle.oracle_run("gemver", inputs, ext, threads=8)
            assert_matches("gemver", run_host("gemver", inputs, ext), want, ext, f"panels {panel_mib} MiB")
            pinned = {k: (torch.from_numpy(v).pin_memory().numpy() if isinstance(v, np.ndarray) else v)
                      for k, v in inputs.items()}
            assert_matches("gemver", run_host("gemver", pinned, ext), want, ext, "pinned")
        for panel_mib, k in ((1, 5000001), (4, 1 << 22), (256, (1 << 22) + 2)):
            _native.set_tuning(host_pipeline=1, host_panel_mib=panel_mib)
            g = bto.load_graph("axpydot")
            inputs = bto.gen_inputs(g, {"M": k}, seed=k % 97)
            want = oracle.oracle_run("axpydot", inputs, {"M": k}, threads=8)
            assert_matches("axpydot", run_host("axpydot", inputs, {"M": k}), want, {"M": k},
                           f"chunks {panel_mib} MiB")
        _native.set_tuning(host_pipeline=0)
        ext = {"M": 2100, "N": 2050}
        g = bto.load_graph("gemver")
        inputs = bto.gen_inputs(g, ext, seed=1)
        assert_matches("gemver", run_host("gemver", inputs, ext),
                       oracle.oracle_run("gemver", inputs, ext, threads=8), ext, "unpipelined")
    finally:
        _native.set_tuning(host_pipeline=1, host_panel_mib=64)


def test_pageable_host_operands_bounce(bto_lib, oracle):
    """Pageable (numpy) operands of 16 MiB and more travel through the pinned bounce
    slots, filled and drained by host threads: one chunk, several chunks, more chunks
    than slots, every thread count, and the direct path with the slots switched off."""
    try:
        for threads, panel_mib, (m, n) in ((0, 256, (1500, 1450)), (1, 256, (3100, 3000)),
                                           (5, 32, (5300, 5200)), (12, 16, (2048, 4096)),
                                           (3, 256, (5300, 5200))):
            _native.set_tuning(host_bounce=1, host_threads=threads, host_panel_mib=panel_mib)
            ext = {"M": m, "N": n}
            for name in ("gemver", "bicgk", "gesummv"):
                g = bto.load_graph(name)
                inputs = bto.gen_inputs(g, ext, seed=n)
                want = oracle.oracle_run(name, inputs, ext, threads=8)
                assert_matches(name, run_host(name, inputs, ext), want, ext, f"bounce, {threads} threads")
        _native.set_tuning(host_bounce=0)
        ext = {"M": 3100, "N": 3000}
        g = bto.load_graph("gemver")
        inputs = bto.gen_inputs(g, ext, seed=2)
        assert_matches("gemver", run_host("gemver", inputs, ext),
                       oracle.oracle_run("gemver", inputs, ext, threads=8), ext, "no bounce")
    finally:
        _native.set_tuning(host_bounce=1, host_threads=0, host_panel_mib=64)


def test_reference_style_ctypes_binding(bto_lib, oracle):
    """Bind the library the way the reference's loader does (runtime.py:99-150):
    raw CDLL, symbol by kernel name, POINTER(c_double) numpy buffers, c_double
    scalars, c_long extents, restype None, NaN-prefilled outputs."""
    import ctypes
    lib = ctypes.CDLL(str(bto.library_path()))
    g = bto.load_graph("gemver")
    ext = {"M": 123, "N": 310}
    inputs = bto.gen_inputs(g, ext, seed=4)
    fn = getattr(lib, g.spec.name.lower())
    fn.restype = None
    dp = ctypes.POINTER(ctypes.c_double)
    args, keep, outs = [], [], {}
    for name, decl in g.spec.inputs:
        if decl.kind == "scalar":
            args.append(ctypes.c_double(inputs[name]))
        else:
            flat = np.ascontiguousarray(inputs[name].ravel())
            keep.append(flat)
            args.append(flat.ctypes.data_as(dp))
    for name, decl in g.spec.outputs:
        buf = np.full(int(np.prod([ext[d] for d in g.dims[name]])), np.nan)
        outs[name] = buf
        args.append(buf.ctypes.data_as(dp))
    args += [ctypes.c_long(ext[e]) for e in g.extent_names]
    fn(*args)
    assert lib.bto_last_error() == 0
    got = {n: outs[n].reshape([ext[d] for d in g.dims[n]]) for n in outs}
    assert_matches("gemver", got, oracle.oracle_run("gemver", inputs, ext, threads=8), ext)


def test_known_answers_on_gpu(bto_lib):
    # the reference's own KATs (tests/test_codegen.py:46-59)
    out = run_host("batax", {"A": np.eye(3), "x": np.array([1.0, 2.0, 3.0]), "beta": 2.0},
                   {"M": 3, "N": 3})
    np.testing.assert_array_equal(out["y"], [2.0, 4.0, 6.0])
    y = np.array([3.0, -1.0, 4.0])
    out = run_host("dgemv", {"A": np.ones((3, 2)), "x": np.ones(2), "alpha": 0.0, "beta": 1.0,
                             "y": y}, {"M": 3, "N": 2})
    np.testing.assert_array_equal(out["z"], y)


# ---- full BASELINE sizes: size-independent properties (no CPU oracle at 8 GiB) ----

def _rand(shape, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    return torch.rand(shape, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1


def _run(name, inputs, ext):
    g = bto.load_graph(name)
    return bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, inputs, ext)


def _err(a, b):
    return float(torch.max(torch.abs(a - b) / torch.clamp(torch.abs(b), min=1.0)))


def test_bench_size_cross_kernel_identities(bto_lib):
    n = 32768
    ext = {"M": n, "N": n}
    t = 1e-12 * math.log2(n)
    A = _rand((n, n), 1)
    p, r = _rand((n,), 2), _rand((n,), 3)
    bi = _run("bicgk", {"A": A, "p": p, "r": r}, ext)
    # independent check of both products (cuBLAS fp64 as a second opinion)
    assert _err(bi["q"], torch.mv(A, p)) <= t
    assert _err(bi["s"], torch.mv(A.t(), r)) <= t
    # ATAX(A, x) == s of BiCGK(A, p=x, r=A x)
    at = _run("atax", {"A": A, "x": p}, ext)
    s2 = _run("bicgk", {"A": A, "p": p, "r": bi["q"]}, ext)["s"]
    assert _err(at["y"], s2) <= t * 4
    # GEMVER with zero rank-2 vectors: B == A bit for bit, x = beta A'y + z, w = alpha A x
    zero = torch.zeros(n, dtype=torch.float64, device="cuda")
    z = _rand((n,), 4)
    ge = _run("gemver", {"A": A, "u1": zero, "v1": zero, "u2": zero, "v2": zero,
                         "alpha": 0.5, "beta": -0.25, "y": r, "z": z}, ext)
    assert torch.equal(ge["B"], A)
    assert _err(ge["x"], -0.25 * bi["s"] + z) <= t
    assert _err(ge["w"], 0.5 * torch.mv(A, ge["x"])) <= t * 4
    # full GEMVER: rows of B against the definition on a sample, x/w via cuBLAS on B
    u1, v1, u2, v2 = (_rand((n,), s) for s in (5, 6, 7, 8))
    ge = _run("gemver", {"A": A, "u1": u1, "v1": v1, "u2": u2, "v2": v2,
                         "alpha": 0.7, "beta": 0.3, "y": r, "z": z}, ext)
    rows = torch.tensor([0, 1, 4097, n // 2, n - 1], device="cuda")
    want = (A[rows] + u1[rows, None] * v1[None, :]) + u2[rows, None] * v2[None, :]
    assert torch.equal(ge["B"][rows], want)
    assert _err(ge["x"], 0.3 * torch.mv(ge["B"].t(), r) + z) <= t
    assert _err(ge["w"], 0.7 * torch.mv(ge["B"], ge["x"])) <= t * 4
    del ge, A, want
    torch.cuda.empty_cache()
    # GESUMMV at its own bench size: B = A and beta = alpha  =>  y = 2 alpha A x
    m = 24576
    A = _rand((m, m), 9)
    x = _rand((m,), 10)
    y = _run("gesummv", {"alpha": 0.375, "beta": 0.375, "A": A, "B": A, "x": x},
             {"M": m, "N": m})["y"]
    assert _err(y, 0.75 * torch.mv(A, x)) <= 1e-12 * math.log2(m)


@pytest.mark.parametrize("shape", [(3, 200001), (2, 2200000), (9, 70000), (300000, 6), (70001, 33), (1, 600000),
                                   (500000, 1), (100000, 2), (40000, 64), (30011, 100), (20000, 255),
                                   (20000, 256), (20000, 257), (5, 256), (77, 130), (9000, 17), (9000, 300), (8000, 511),
                                   (8000, 512), (4000, 514), (3000, 390)])
def test_extreme_aspect_ratios(bto_lib, oracle, shape):
    """Short-wide matrices have thousands of column strips (the row-side join then shares a
    row between a warp or a whole CTA); tall-skinny ones (N <= 256) take skinny_kernels.cuh,
    where L threads share a row -- checked with that path on and off."""
    m, n = shape
    try:
        for skinny in ((1, 0) if n <= 512 else (1,)):
            _native.set_tuning(skinny=skinny)
            for name in ("bicgk", "atax", "gesummv", "gemver", "dgemv", "dgemvt", "batax"):
                ext = ext_of(name, m, n)
                graph = bto.load_graph(name)
                inputs = bto.random_inputs(graph, ext, seed=m % 13)
                want = oracle.oracle_run(name, inputs, ext, threads=4)
                assert_matches(name, run_device(name, inputs, ext), want, ext, f"aspect ratio, skinny={skinny}")
    finally:
        _native.set_tuning(skinny=1)


@pytest.mark.parametrize("shape", [(2, 2200000), (8, 700000), (64, 650000), (20, 1000002), (1, 620000),
                                   (130, 610000)])
def test_short_wide_matrices_finish_columns_in_the_producer(bto_lib, oracle, shape):
    """Thousands of strips, a few units each: CTAs take whole strips and apply the column
    epilogue themselves (mv_tile_direct_kernel) -- no column partials, no column join.  Same
    results as the partial + join path up to the order of the row-unit sums (identical here:
    a strip's column sum is accumulated by one thread in ascending row order either way)."""
    m, n = shape
    ext = {"M": m, "N": n}
    try:
        for name in ("bicgk", "gemver", "dgemvt", "atax", "batax"):
            graph = bto.load_graph(name)
            inputs = bto.gen_inputs(graph, ext, seed=m + n)
            want = oracle.oracle_run(name, inputs, ext, threads=8)
            if name in ("atax", "batax"):
                # t = A x sums up to 10^6 cancelling terms; the oracle adds them one after the other
                # (as the reference's C does) and is itself ~5e-11 off at N = 700000, the GPU's tree
                # order ~1e-12: check these two against an extended-precision evaluation instead
                A, x = inputs["A"].astype(np.longdouble), inputs["x"].astype(np.longdouble)
                y = A.T @ (A @ x)
                if name == "batax":
                    y = y * np.longdouble(inputs["beta"])
                assert bto.max_rel_error({"y": want["y"]}, {"y": y.astype(np.float64)}) < 1e-9   # same function
                want = {"y": y.astype(np.float64)}
            plans = {}
            for direct in (1, 0):
                _native.set_tuning(direct_cols=direct)
                got = run_device(name, inputs, ext)
                plans[direct] = _native.launch_plan()
                assert_matches(name, got, want, ext, f"direct_cols={direct}")
            assert "mv_tile_direct_kernel" in plans[1] and "direct" not in plans[0], plans
    finally:
        _native.set_tuning(direct_cols=1)


@pytest.mark.parametrize("shape", [(600, 4096), (1001, 4098), (593, 6002), (2500, 9000), (4097, 4100)])
def test_gesummv_row_streaming(bto_lib, oracle, shape):
    """Wide GESUMMV streams whole rows (rowstream_kernels.cuh) instead of column strips: one
    launch, no partials; checked against the oracle with that path on and off."""
    m, n = shape
    g = bto.load_graph("gesummv")
    ext = {"M": m, "N": n}
    inputs = bto.random_inputs(g, ext, seed=n)
    want = oracle.oracle_run("gesummv", inputs, ext, threads=8)
    try:
        for on in (1, 0):
            _native.set_tuning(rowstream=on)
            before = _native.kernel_launches()
            got = run_device("gesummv", inputs, ext)
            assert _native.kernel_launches() - before == (1 if on else 2)
            assert_matches("gesummv", got, want, ext, f"rowstream={on}")
        # x at an odd 8-byte offset next to 16-byte-aligned matrices
        dev = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in inputs.items()}
        shifted = torch.empty(n + 1, dtype=torch.float64, device="cuda")[1:]
        shifted.copy_(dev["x"])
        assert shifted.data_ptr() % 16 == 8
        dev["x"] = shifted
        out = bto.run_kernel(bto.library_path(), bto.gpu_kernel(g), g, dev, ext)
        assert_matches("gesummv", {k: v.cpu().numpy() for k, v in out.items()}, want, ext, "misaligned x")
    finally:
        _native.set_tuning(rowstream=1)


def test_column_major_corpus_kernels_stay_fused(bto_lib, oracle):
    """`matrix(column)` operands: the same logical kernel, the
    buffers are F-ordered.  The library maps every corpus sequence onto its row-major fused
    passes with the products' roles swapped (colmajor.py); results equal the row-major
    oracle on the same logical matrices, B bit for bit."""
    from paper_1205_1098_b200 import spec as bspec
    for name in ("bicgk", "atax", "batax", "gesummv", "dgemv", "dgemvt", "gemver"):
        text = bspec.CORPUS[name].replace("matrix(row)", "matrix(column)")
        graph = bspec.infer_shapes(bspec.parse_kernel(text))
        kernel = bto.gpu_kernel(graph, allow_generic=False)
        assert kernel.source == f"libbto_b200:colmajor:{name}"
        row_graph = bto.load_graph(name)
        for (m, n) in ((1, 1), (5, 3), (130, 257), (1025, 700), (2048, 2048), (600, 4100)):
            ext = ext_of(name, m, n)
            inputs = bto.random_inputs(row_graph, ext, seed=m + n)
            want = oracle.oracle_run(name, inputs, ext, threads=4)
            # numpy in (C-ordered logical arrays, as a caller would hold them) -> numpy out
            got = bto.run_kernel(bto.library_path(), kernel, graph, inputs, ext)
            assert_matches(name, got, want, ext, "column-major, numpy")
            # F-ordered CUDA tensors are used in place and B comes back F-ordered
            dev = {k: (torch.from_numpy(np.asfortranarray(v)).cuda() if isinstance(v, np.ndarray) else v)
                   for k, v in inputs.items()}
            before = _native.kernel_launches()
            out = bto.run_kernel(bto.library_path(), kernel, graph, dev, ext)
            launches = _native.kernel_launches() - before
            assert launches <= {"bicgk": 2, "gemver": 4, "dgemv": 3}.get(name, 4), (name, launches)
            assert_matches(name, {k: v.cpu().numpy() for k, v in out.items()}, want, ext,
                           "column-major, device")
            if name == "gemver" and m > 1 and n > 1:
                assert out["B"].t().is_contiguous()


def test_more_than_2_to_the_32_elements(bto_lib):
    """Matrices of 4.3e9 and more elements (32-36 GiB each): every index computation has to
    be 64-bit.  Rank-1 matrices A = a b' give closed forms at any size:
    A p = a (b.p), A' r = b (a.r), A'(A x) = b (a.a)(b.x)."""
    free, _ = torch.cuda.mem_get_info()
    if free < 100 * 2 ** 30:
        pytest.skip("needs ~80 GiB of free HBM")

    def rank1(m, n, seed):
        a, b = _rand((m,), seed), _rand((n,), seed + 1)
        A = torch.empty((m, n), dtype=torch.float64, device="cuda")
        torch.outer(a, b, out=A)
        return A, a, b

    def close(got, want, scale, tol):
        return float(torch.max(torch.abs(got - want))) <= tol * scale

    for m, n in ((65536, 65536), (36000, 120000)):
        ext = {"M": m, "N": n}
        A, a, b = rank1(m, n, m % 97)
        p, r = _rand((n,), 3), _rand((m,), 4)
        bp, ar, aa = float(torch.dot(b, p)), float(torch.dot(a, r)), float(torch.dot(a, a))
        scale = math.sqrt(max(m, n))                     # size of a length-n dot of U[-1,1) terms
        out = _run("bicgk", {"A": A, "p": p, "r": r}, ext)
        assert close(out["q"], a * bp, scale, 1e-12) and close(out["s"], b * ar, scale, 1e-12)
        y = _run("atax", {"A": A, "x": p}, ext)["y"]
        want = b * (aa * bp)
        assert close(y, want, float(torch.max(torch.abs(want))), 1e-11)
        # the last row / column really were read: perturb one corner element
        A[m - 1, n - 1] += 1.0
        out2 = _run("bicgk", {"A": A, "p": p, "r": r}, ext)
        assert abs(float(out2["q"][m - 1] - out["q"][m - 1]) - float(p[n - 1])) <= 1e-9
        assert abs(float(out2["s"][n - 1] - out["s"][n - 1]) - float(r[m - 1])) <= 1e-9
        assert torch.equal(out2["q"][: m - 1], out["q"][: m - 1])
        del out, out2, y
        if m == n:
            # GEMVER with A and B of 32 GiB each: sampled rows of B bit-exact, x and w closed-form
            u1, v1, u2, v2, yv, z = (_rand((n,), sd) for sd in (5, 6, 7, 8, 9, 10))
            A[m - 1, n - 1] -= 1.0
            ge = _run("gemver", {"A": A, "u1": u1, "v1": v1, "u2": u2, "v2": v2,
                                 "alpha": 0.7, "beta": 0.3, "y": yv, "z": z}, ext)
            rows = torch.tensor([0, 1, 32767, 32768, m - 1], device="cuda")
            want = (A[rows] + u1[rows, None] * v1[None, :]) + u2[rows, None] * v2[None, :]
            assert torch.equal(ge["B"][rows], want)
            bty = b * float(torch.dot(a, yv)) + v1 * float(torch.dot(u1, yv)) + v2 * float(torch.dot(u2, yv))
            assert close(ge["x"], 0.3 * bty + z, scale, 1e-11)
            x = ge["x"]
            bx = a * float(torch.dot(b, x)) + u1 * float(torch.dot(v1, x)) + u2 * float(torch.dot(v2, x))
            assert close(ge["w"], 0.7 * bx, float(torch.max(torch.abs(bx))), 1e-11)
            del ge, want
        del A
        torch.cuda.empty_cache()
    # GESUMMV: two matrices of 2^32 + elements would need 69 GiB; 50000^2 x 2 = 40 GB is the same code path
    m = 50000
    A, a, b = rank1(m, m, 11)
    B, c, d = rank1(m, m, 13)
    x = _rand((m,), 15)
    y = _run("gesummv", {"alpha": 0.375, "beta": -0.5, "A": A, "B": B, "x": x}, {"M": m, "N": m})["y"]
    want = 0.375 * a * float(torch.dot(b, x)) - 0.5 * c * float(torch.dot(d, x))
    assert close(y, want, math.sqrt(m), 1e-12)
    # AXPYDOT on 2^32 + 5 elements (4 vectors of 32 GiB)
    del A, B
    torch.cuda.empty_cache()
    k = (1 << 32) + 5
    w = torch.empty(k, dtype=torch.float64, device="cuda")
    w[: 1 << 31] = _rand((1 << 31,), 17)
    w[1 << 31: 1 << 32] = w[: 1 << 31]
    w[1 << 32:] = 3.0
    out = _run("axpydot", {"w": w, "v": w, "u": w, "alpha": 0.5}, {"M": k})
    assert torch.equal(out["z"][-5:], torch.full((5,), 1.5, dtype=torch.float64, device="cuda"))
    assert torch.equal(out["z"][: 1 << 20], w[: 1 << 20] - w[: 1 << 20] * 0.5)
    q4 = 1 << 30                                              # (torch.dot takes < 2^31 elements)
    half = float(torch.dot(w[:q4], w[:q4])) + float(torch.dot(w[q4: 2 * q4], w[q4: 2 * q4]))  # beta = 0.5 * sum w^2
    assert abs(out["beta"] - (0.5 * (2 * half + 45.0))) <= 1e-10 * half


def test_bench_size_axpydot_properties(bto_lib):
    n = 1 << 27
    w, v, u = _rand((n,), 1), _rand((n,), 2), _rand((n,), 3)
    out = _run("axpydot", {"w": w, "v": v, "u": u, "alpha": 0.0}, {"M": n})
    assert torch.equal(out["z"], w)                      # alpha = 0: z is w, bit for bit
    ref = float(torch.dot(w, u))
    assert abs(out["beta"] - ref) / max(abs(ref), 1.0) <= 1e-12 * 27
    out = _run("axpydot", {"w": w, "v": v, "u": u, "alpha": -0.625}, {"M": n})
    assert torch.equal(out["z"], w - v * (-0.625))       # mul then sub, each rounded once
    ref = float(torch.dot(out["z"], u))
    assert abs(out["beta"] - ref) / max(abs(ref), 1.0) <= 1e-12 * 27


def test_random_extents_like_reference_criterion_1(bto_lib, oracle):
    """The reference's acceptance criterion 1 (tests/test_acceptance.py:55-94) walks
    every kernel over a grid of extents; here 40 seeded random extent pairs per
    kernel, including degenerate ones, against the live oracle."""
    rng = np.random.default_rng(20121205)
    for name in KERNELS:
        graph = bto.load_graph(name)
        pairs = [(1, 1), (2, 2), (1, 7), (7, 1)]
        pairs += [(int(rng.integers(1, 700)), int(rng.integers(1, 3000))) for _ in range(18)]
        pairs += [(int(rng.integers(1, 3000)), int(rng.integers(1, 700))) for _ in range(18)]
        for idx, (m, n) in enumerate(pairs):
            ext = ext_of(name, m, n)
            inputs = bto.random_inputs(graph, ext, seed=idx)
            want = oracle.oracle_run(name, inputs, ext, threads=1 + idx % 8)
            assert_matches(name, run_device(name, inputs, ext), want, ext, "random extents")


def test_cuda_graph_capture_and_replay(bto_lib, oracle):
    """The asynchronous entry points are stream-ordered and allocation-free after a
    warm-up call, so a whole sequence can be captured into a CUDA graph (what the
    sharded runtime does to hide launch gaps) and replayed on new data."""
    from paper_1205_1098_b200.sharded import GpuShardOps
    m, n = 1536, 2048
    g = bto.load_graph("gemver")
    inputs = bto.gen_inputs(g, {"M": m, "N": n}, seed=3)
    dev = {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in inputs.items()}
    B = torch.empty(m, n, dtype=torch.float64, device="cuda")
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    w = torch.empty(m, dtype=torch.float64, device="cuda")
    ops = GpuShardOps()

    def launch():
        ops.gemver(dev["A"], dev["u1"], dev["v1"], dev["u2"], dev["v2"], inputs["alpha"],
                   inputs["beta"], dev["y"], dev["z"], B, x, w)

    launch()                       # warm-up: sizes the workspace outside the capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        launch()
    # new data in the same buffers, then replay
    inputs2 = bto.gen_inputs(g, {"M": m, "N": n}, seed=4)
    inputs2["alpha"], inputs2["beta"] = inputs["alpha"], inputs["beta"]   # scalars are baked in
    for k, v in inputs2.items():
        if isinstance(v, np.ndarray):
            dev[k].copy_(torch.from_numpy(v))
    B.fill_(float("nan")); x.fill_(float("nan")); w.fill_(float("nan"))
    graph.replay()
    torch.cuda.synchronize()
    want = oracle.oracle_run("gemver", inputs2, {"M": m, "N": n}, threads=8)
    got = {"B": B.cpu().numpy(), "x": x.cpu().numpy(), "w": w.cpu().numpy()}
    assert_matches("gemver", got, want, {"M": m, "N": n}, "graph replay")


def test_two_streams_run_concurrently_without_sharing_partials(bto_lib, oracle):
    """Every stream has its own partial-sum workspace and ticket counters (include/bto_b200.h
    section 2): BiCGK, ATAX and AXPYDOT enqueued on two streams at once, 1000 rounds, with
    different shapes per stream so that one stream's partials could never pass for the
    other's.  Until round 2 there was one workspace per device and this returned wrong sums."""
    from paper_1205_1098_b200.sharded import GpuShardOps
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    shapes = [(1200, 2300), (900, 3100)]
    cases = []
    for st, (m, n) in zip(streams, shapes):
        ext = {"M": m, "N": n}
        gb, ga, gx = bto.load_graph("bicgk"), bto.load_graph("atax"), bto.load_graph("axpydot")
        ib, ia = bto.gen_inputs(gb, ext, seed=m), bto.gen_inputs(ga, ext, seed=n)
        ix = bto.gen_inputs(gx, {"M": m * 97}, seed=m + n)
        dev = lambda d: {k: (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray) else v) for k, v in d.items()}
        case = {"ops": GpuShardOps(stream=st), "ext": ext, "ib": dev(ib), "ia": dev(ia), "ix": dev(ix),
                "want_b": oracle.oracle_run("bicgk", ib, ext, threads=8),
                "want_a": oracle.oracle_run("atax", ia, ext, threads=8),
                "want_x": oracle.oracle_run("axpydot", ix, {"M": m * 97}, threads=8),
                "q": torch.empty(m, dtype=torch.float64, device="cuda"),
                "s": torch.empty(n, dtype=torch.float64, device="cuda"),
                "y": torch.empty(n, dtype=torch.float64, device="cuda"),
                "z": torch.empty(m * 97, dtype=torch.float64, device="cuda"),
                "beta": torch.empty(1, dtype=torch.float64, device="cuda")}
        cases.append(case)
    torch.cuda.synchronize()
    first = None
    for rnd in range(1000):
        for c in cases:
            for t in (c["q"], c["s"], c["y"], c["beta"]):
                with torch.cuda.stream(c["ops"]._stream):
                    t.fill_(float("nan"))
        for c in cases:                         # interleaved issue: both streams stay busy
            c["ops"].bicgk(c["ib"]["A"], c["ib"]["p"], c["ib"]["r"], c["q"], c["s"])
        for c in cases:
            c["ops"].atax(c["ia"]["A"], c["ia"]["x"], c["y"])
        for c in cases:
            c["ops"].axpydot(c["ix"]["w"], c["ix"]["v"], c["ix"]["u"], c["ix"]["alpha"], c["z"], c["beta"])
        torch.cuda.synchronize()
        snap = [torch.cat([c["q"], c["s"], c["y"], c["beta"]]).clone() for c in cases]
        if first is None:
            first = snap
            for c in cases:
                assert_matches("bicgk", {"q": c["q"].cpu().numpy(), "s": c["s"].cpu().numpy()}, c["want_b"], c["ext"])
                assert_matches("atax", {"y": c["y"].cpu().numpy()}, c["want_a"], c["ext"])
                assert_matches("axpydot", {"z": c["z"].cpu().numpy(), "beta": float(c["beta"][0])}, c["want_x"],
                               {"M": c["ext"]["M"] * 97})
        else:                                   # fixed reduction order: every round the same bits
            for a, b in zip(first, snap):
                assert torch.equal(a, b), f"round {rnd}: results changed under concurrency"


def test_captured_graph_survives_workspace_growth(bto_lib, oracle):
    """A graph captured on a stream keeps replaying correctly after a LARGER call on the same
    stream made the workspace grow (the chunk a captured kernel uses is retired, not freed), and
    growth during capture itself is legal."""
    from paper_1205_1098_b200.sharded import GpuShardOps
    st = torch.cuda.Stream()
    ops = GpuShardOps(stream=st)
    g = bto.load_graph("bicgk")
    small, large = {"M": 1500, "N": 2100}, {"M": 9000, "N": 7000}
    ins = {tag: bto.gen_inputs(g, ext, seed=9) for tag, ext in (("small", small), ("large", large))}
    dev = {tag: {k: torch.from_numpy(v).cuda() for k, v in d.items()} for tag, d in ins.items()}
    out = {tag: (torch.empty(ext["M"], dtype=torch.float64, device="cuda"),
                 torch.empty(ext["N"], dtype=torch.float64, device="cuda"))
           for tag, ext in (("small", small), ("large", large))}
    torch.cuda.synchronize()
    before = _native.load().bto_workspace_bytes()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):     # first call on this stream: it allocates under capture
        ops.bicgk(dev["small"]["A"], dev["small"]["p"], dev["small"]["r"], *out["small"])
    assert _native.load().bto_workspace_bytes() > before
    with torch.cuda.stream(st):
        ops.bicgk(dev["large"]["A"], dev["large"]["p"], dev["large"]["r"], *out["large"])   # grows
    torch.cuda.synchronize()
    for t in out["small"]:
        t.fill_(float("nan"))
    torch.cuda.synchronize()
    graph.replay()
    torch.cuda.synchronize()
    for tag, ext in (("small", small), ("large", large)):
        want = oracle.oracle_run("bicgk", ins[tag], ext, threads=8)
        assert_matches("bicgk", {"q": out[tag][0].cpu().numpy(), "s": out[tag][1].cpu().numpy()}, want, ext, tag)
    # an explicit reservation makes later calls allocation-free
    _native.check(_native.load().bto_reserve_workspace(st.cuda_stream, 64 << 20))
    held = _native.load().bto_workspace_bytes()
    with torch.cuda.stream(st):
        ops.bicgk(dev["large"]["A"], dev["large"]["p"], dev["large"]["r"], *out["large"])
    assert _native.load().bto_workspace_bytes() == held


@pytest.mark.parametrize("name", KERNELS)
def test_no_write_lands_outside_the_outputs(bto_lib, oracle, name):
    """compute-sanitizer is closed on this GPU pool (gpurun answers so), so out-of-bounds WRITES are
    hunted with guard bands: every operand lives inside one arena, separated by canary words with
    a recognisable bit pattern; after each call the canaries and the inputs must be bit-identical
    and the outputs must match the oracle.  Ragged and unaligned shapes, every launch path
    (strip tiles, shared-row kernels, whole-row streaming, cluster ATAX, the two-pass fallback)."""
    graph = bto.load_graph(name)
    kernel = bto.gpu_kernel(graph)
    canary = float(np.frombuffer(np.uint64(0x7FF8DEADBEEF1234).tobytes(), dtype=np.float64)[0])
    shapes = RAGGED + [(2048, 1024), (600, 4100), (37, 16390), (4100, 300), (5, 70001)]
    for pad in (2, 3):                   # even / odd guard widths: 16-byte aligned and 8-byte-offset operands
        for (m, n) in shapes:
            ext = ext_of(name, m, n)
            inputs = bto.gen_inputs(graph, ext, seed=m + 3 * n)
            want = oracle.oracle_run(name, inputs, ext, threads=8)
            sizes = []
            for pname, decl in graph.spec.inputs + graph.spec.outputs:
                if (pname, decl) in graph.spec.inputs and decl.kind == "scalar":
                    continue
                count = 1
                for d in graph.dims[pname]:
                    count *= int(ext[d])
                sizes.append((pname, count))
            total = pad + sum(c + pad for _, c in sizes)
            arena = torch.full((total,), canary, dtype=torch.float64, device="cuda")
            views, off = {}, pad
            for pname, count in sizes:
                views[pname] = arena[off:off + count]
                off += count + pad
            dev_in, outs = {}, {}
            for pname, decl in graph.spec.inputs:
                if decl.kind == "scalar":
                    dev_in[pname] = inputs[pname]
                else:
                    views[pname].copy_(torch.from_numpy(np.ascontiguousarray(inputs[pname]).ravel()))
                    dev_in[pname] = views[pname].view(tuple(int(ext[d]) for d in graph.dims[pname]))
            for pname, decl in graph.spec.outputs:
                views[pname].fill_(float("nan"))
                outs[pname] = views[pname]
            before = arena.clone()
            bto.run_kernel_async(kernel, graph, dev_in, ext, outs)
            torch.cuda.synchronize()
            # everything except the outputs is bit-identical to before the call
            mask = torch.ones(total, dtype=torch.bool, device="cuda")
            off = pad
            for pname, count in sizes:
                if any(pname == o for o, _ in graph.spec.outputs):
                    mask[off:off + count] = False
                off += count + pad
            same = arena.view(torch.int64)[mask] == before.view(torch.int64)[mask]
            assert bool(same.all()), f"{name} {ext} pad {pad}: wrote outside its outputs"
            got = {o: (float(outs[o][0]) if d.kind == "scalar" else
                       outs[o].view(tuple(int(ext[x]) for x in graph.dims[o])).cpu().numpy())
                   for o, d in graph.spec.outputs}
            assert_matches(name, got, want, ext, f"guard bands, pad {pad}")


def test_randomised_differential_run(bto_lib, oracle):
    """20 s of tests/fuzz_parity.py: random kernels, extents biased to tile / strip edges, random
    launch tunables, host and device operands, all against the oracle."""
    import subprocess, sys
    from pathlib import Path
    script = Path(__file__).with_name("fuzz_parity.py")
    proc = subprocess.run([sys.executable, str(script), "20", "1205"], capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-2000:]
    assert " 0 mismatches" in proc.stdout


def test_staged_host_copies_round_trip(bto_lib):
    """bto_copy_to_device / bto_copy_to_host: below and above the bounce threshold, more chunks
    than slots, non-contiguous input, pinned memory."""
    rng = np.random.default_rng(5)
    for shape in ((1,), (1000, 3), (2 * 1024 * 1024 + 1,), (3001, 3001), (6000, 5000)):
        a = rng.uniform(-1, 1, size=shape)
        t = _native.to_device(a)
        assert tuple(t.shape) == shape and torch.equal(t.cpu(), torch.from_numpy(a))
        assert np.array_equal(_native.to_host(t), a)
    a = rng.uniform(-1, 1, size=(2500, 2600))
    assert np.array_equal(_native.to_host(_native.to_device(a.T)), a.T)          # strided view in
    p = torch.from_numpy(a).pin_memory().numpy()
    assert np.array_equal(_native.to_host(_native.to_device(p)), a)


def test_bound_calls_replay(bto_lib, oracle):
    """GpuShardOps.bind pre-marshals a call; replaying it on new data in the same buffers gives
    the results of a fresh call."""
    from paper_1205_1098_b200.sharded import GpuShardOps
    ops = GpuShardOps()
    m, n = 700, 1300
    g = bto.load_graph("gemver")
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    first = bto.gen_inputs(g, {"M": m, "N": n}, seed=1)
    bufs = {k: dev(v) for k, v in first.items() if isinstance(v, np.ndarray)}
    B, x, w = (torch.full(s, float("nan"), dtype=torch.float64, device="cuda") for s in ((m, n), (n,), (m,)))
    call = ops.bind("gemver", bufs["A"], bufs["u1"], bufs["v1"], bufs["u2"], bufs["v2"], first["alpha"],
                    first["beta"], bufs["y"], bufs["z"], B, x, w)
    for seed in (1, 2, 3):
        inputs = bto.gen_inputs(g, {"M": m, "N": n}, seed=seed)
        inputs["alpha"], inputs["beta"] = first["alpha"], first["beta"]      # scalars are part of the binding
        for k, t in bufs.items():
            t.copy_(dev(inputs[k]))
        call()
        torch.cuda.synchronize()
        want = oracle.oracle_run("gemver", inputs, {"M": m, "N": n}, threads=4)
        assert_matches("gemver", {"B": B.cpu().numpy(), "x": x.cpu().numpy(), "w": w.cpu().numpy()}, want,
                       {"M": m, "N": n}, f"bound call, seed {seed}")


@pytest.mark.parametrize("shape", [(1030, 2050), (4001, 130)], ids=["tiles", "shared-rows"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_join_fused_exchange_emulated_ranks(bto_lib, oracle, world, shape):
    """The join kernel that does the cross-GPU all-reduce itself (peer-memory one-shot,
    include/bto_b200.h 3b), with ONE GPU standing in for all ranks: the exchange
    buffers and flag arrays of every "rank" live on this device; first every rank
    runs its sequence with exchange_phases=1 (join + publish), then every rank with
    exchange_phases=2 (wait -- already satisfied -- + rank-ordered reduce).  No kernel
    ever waits on another, so this is safe on one device, and it covers the index
    math, the flag protocol and the rank-ordered sum; only the concurrency of real
    peers is not exercised."""
    import ctypes
    from paper_1205_1098_b200.sharded import GpuShardOps, row_block, shard_inputs
    lib = _native.load()
    ops = GpuShardOps()
    m, n = shape
    capacity = 2 * max(m, n)
    exch = [torch.zeros(capacity, dtype=torch.float64, device="cuda") for _ in range(world)]
    flags = [torch.zeros(lib.bto_exchange_flag_bytes(world) // 4, dtype=torch.int32, device="cuda")
             for _ in range(world)]
    exch_ptrs = (ctypes.c_void_p * world)(*[t.data_ptr() for t in exch])
    flag_ptrs = (ctypes.c_void_p * world)(*[t.data_ptr() for t in flags])
    epoch = 0
    try:
        for name in ("bicgk", "atax", "gemver", "axpydot"):
            graph = bto.load_graph(name)
            ext = {"M": m} if name == "axpydot" else {"M": m, "N": n}
            full = bto.gen_inputs(graph, ext, seed=bto.SEEDS[name])
            want = oracle.oracle_run(name, full, ext, threads=8)
            outs = []
            for r in range(world):
                lo, hi = row_block(m, r, world)
                mine = {k: (torch.from_numpy(np.ascontiguousarray(v)).cuda() if isinstance(v, np.ndarray) else v)
                        for k, v in shard_inputs(name, full, r, world, m).items()}
                nan = lambda *shape: torch.full(shape, float("nan"), dtype=torch.float64, device="cuda")
                if name == "bicgk":
                    o = {"q": nan(hi - lo), "s": nan(n)}
                    call = lambda t=mine, o=o: ops.bicgk_sharded(t["A"], t["p"], t["r"], o["q"], o["s"])
                elif name == "atax":
                    o = {"y": nan(n)}
                    call = lambda t=mine, o=o: ops.atax_sharded(t["A"], t["x"], o["y"])
                elif name == "gemver":
                    o = {"B": nan(hi - lo, n), "x": nan(n), "w": nan(hi - lo)}
                    call = lambda t=mine, o=o: ops.gemver_sharded(
                        t["A"], t["u1"], t["v1"], t["u2"], t["v2"], t["alpha"], t["beta"], t["y"],
                        t["z"], o["B"], o["x"], o["w"])
                else:
                    o = {"z": nan(hi - lo), "beta": nan(1)}
                    call = lambda t=mine, o=o: ops.axpydot_sharded(t["w"], t["v"], t["u"], t["alpha"],
                                                                   o["z"], o["beta"])
                outs.append((o, call))
            # the epoch counter lives on the device (one per rank); ONE device stands in for all
            # ranks here, so every emulated rank is re-initialised with the exchanges completed so far
            for phase in (1, 2):
                _native.set_tuning(exchange_phases=phase)
                for r, (o, call) in enumerate(outs):
                    _native.check(lib.bto_exchange_init(r, world, exch_ptrs, flag_ptrs, capacity, epoch))
                    _native.poison_shared_memory()      # (a rank's kernels read only what they wrote)
                    _native.poison_workspace()
                    call()
                    torch.cuda.synchronize()
                    done = ctypes.c_uint(0)
                    _native.check(lib.bto_exchange_status(ctypes.byref(done)))
                    assert done.value == epoch + (1 if phase == 2 else 0)
            epoch += 1
            from paper_1205_1098_b200.sharded import SHARDING
            spec = SHARDING[name]
            got = {}
            for out_name in want:
                if out_name in spec.sharded_out:
                    got[out_name] = torch.cat([o[out_name] for o, _ in outs]).cpu().numpy()
                else:
                    first = outs[0][0][out_name]
                    for o, _ in outs[1:]:
                        assert torch.equal(o[out_name], first), f"{name}.{out_name}: ranks disagree"
                    got[out_name] = first.cpu().numpy() if first.numel() > 1 else float(first[0])
            assert_matches(name, got, want, ext, f"fused exchange, world {world}")
    finally:
        _native.set_tuning(exchange_phases=3)
        _native.check(lib.bto_exchange_shutdown())


def test_bench_suite_shards_cleanly_as_rank_1_of_4(bto_lib, monkeypatch):
    """bench.py's per-rank buffers and launches for N > 1 (rank 1 of 4), with the
    all-reduce stubbed out: exercises the row-block slicing, the views GESUMMV
    borrows, and the split GEMVER path, which a 1-GPU box cannot run under NCCL."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench
    from paper_1205_1098_b200 import sharded

    calls = []

    class FakeComm:
        def all_reduce_sum(self, tensor):
            calls.append(tensor.numel())

    monkeypatch.setattr(sharded, "TorchComm", FakeComm)
    suite = bench.Suite(torch, 1, 4, bench.SUITE)
    assert suite.rows == 8192 and suite.grows == 6144 and suite.an == (1 << 27) // 4
    for name in bench.SUITE:
        suite.launch(name)
    torch.cuda.synchronize()
    assert calls == [1, 32768, 32768, 32768]          # axpydot, bicgk s, atax y, gemver B'y
    for t in (suite.q, suite.s, suite.x, suite.w, suite.gy, suite.az, suite.abeta):
        assert bool(torch.isfinite(t).all())
    # the shard's GEMVER equals the definition on its rows (x replicated)
    want_w = 0.83 * torch.mv(suite.Bm, suite.x)
    assert float(torch.max(torch.abs(suite.w - want_w) / torch.clamp(torch.abs(want_w), min=1.0))) < 1e-11
