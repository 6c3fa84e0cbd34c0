"""bench.py's JSON line against the driver's contract, checked on the committed line of the
round's final run (profiles/r01/bench_v14_final.json) and on the reference arm's code path
(which runs on CPU: the oracle / oracle/_ref, a bounded sample)."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
FINAL = REPO / "profiles" / "r01" / "bench_v14_final.json"


def _line(text: str) -> dict:
    return json.loads(text.strip().splitlines()[-1])


def test_committed_bench_line_has_every_contract_key():
    d = _line(FINAL.read_text())
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "clocks", "gpu_launches"):
        assert key in d, key
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True and d["vs_baseline"] is None
    assert d["dtype"] == "f64" and d["data"] == "synthetic" and d["n_gpus"] == 1
    assert "workload" in d["config"] and "model" not in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert r["traffic"] is None or 0.9 < r["traffic"] / r["algorithmic_bytes"] < 1.1     # no wasted re-reads
    c = d["cpu_baseline"]
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] < d["value"]                      # PCIe-bound: never the device-resident figure
    assert d["gpu_launches"] > 0 and d["steps"] >= 1 and d["warmup"] >= 3
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert not bad & set(d["clocks"]["reasons"])
    # the time-based value is consistent with the per-step time and the suite's algorithmic bytes
    total = sum(v["bytes_min"] for v in d["per_kernel"].values())
    assert abs(d["value"] - total / (d["ms_per_step"] * 1e-3) / 1e9) < 0.01 * d["value"]


def test_reference_arm_runs_on_cpu_and_prints_the_contract_line():
    """`bench.py --impl reference` times the reference's generated C (oracle/_ref) or the oracle
    port on the host cores; one AXPYDOT step of the bounded sample keeps this test short."""
    proc = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--kernel", "axpydot",
                           "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-2000:]
    d = _line(proc.stdout)
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["gpu_launches"] == 0


def test_other_ranks_of_the_reference_arm_exit_without_work():
    import os
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    proc = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--gpus", "2"],
                          capture_output=True, text=True, timeout=120, env=env)
    assert proc.returncode == 0 and proc.stdout.strip() == ""


def test_both_arms_print_the_same_config_object():
    """The driver compares the two arms' `config`; what differs between them (host threads, the
    exchange, the timing method) lives in other keys."""
    sys.path.insert(0, str(REPO))
    import bench
    proc = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--kernel", "axpydot",
                           "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-2000:]
    d = _line(proc.stdout)
    assert d["config"] == bench.config_of(("axpydot",), 1)          # what run_gpu_arm prints
    assert d["warmup"] == 0 and d["steps"] == 1                     # the counts actually used
    assert "2^27" in bench.config_of(bench.SUITE, 1)["workload"]
    assert "REDUCED" in bench.describe(bench.CPU_SAMPLE, bench.SUITE)  # a scaled-down run says so
    u = d["cpu_baseline"].get("unfused")
    if d["cpu_baseline"]["kind"] == "reference":
        assert u and u["cores"] == 1 and u["value"] > 0 and u["fusion_speedup_1_thread"] > 1.0


def test_gpus_n_without_n_devices_fails_loudly(monkeypatch):
    """`python bench.py --gpus 2` launches the ranks itself; with fewer than 2 GPUs visible it must
    say so and exit non-zero, not run on one GPU (it printed n_gpus = 1)."""
    import os
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    import torch
    if torch.cuda.is_available() and torch.cuda.device_count() >= 2:
        pytest.skip("two GPUs visible: the spawn path is covered by the multi-GPU test")
    proc = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--steps", "1", "--no-e2e",
                           "--no-cpu"], capture_output=True, text=True, timeout=300, env=env)
    assert proc.returncode != 0
    d = _line(proc.stdout)
    assert "error" in d and d["n_gpus_requested"] == 2 and d["n_gpus_visible"] < 2
    # under a launcher whose world size disagrees with --gpus: refuse as well
    env2 = dict(env, WORLD_SIZE="4", RANK="0", LOCAL_RANK="0")
    proc = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--steps", "1", "--no-e2e",
                           "--no-cpu"], capture_output=True, text=True, timeout=300, env=env2)
    assert proc.returncode != 0 and "error" in _line(proc.stdout)


def test_traffic_json_is_only_quoted_for_the_kernels_it_profiled():
    sys.path.insert(0, str(REPO))
    import bench
    tj = json.loads((REPO / "profiles" / "traffic.json").read_text())
    names = [bench.normalise_kernel_name(k) for k in tj["gemver"]["kernels"]]
    plan = "+".join([names[0], "finalize_kernel"] + names[1:] + ["finalize_kernel"])
    assert bench.traffic_for("gemver", plan)[0] == tj["gemver"]["dram_bytes"]
    stale, why = bench.traffic_for("gemver", "mv_tile_kernel<12,8,1,1,1>+finalize_kernel")
    assert stale is None and why.startswith("stale")


@pytest.mark.gpu
def test_traffic_json_matches_the_kernels_the_library_launches(bto_lib):
    """profiles/traffic.json (ncu DRAM bytes) must have been captured on the kernel instances the
    library launches at the bench sizes today -- a kernel change without a new capture fails here."""
    import torch
    sys.path.insert(0, str(REPO))
    import bench
    from paper_1205_1098_b200 import _native
    suite = bench.Suite(torch, 0, 1, bench.SUITE)
    for k in bench.SUITE:
        suite.launch(k)
        plan = _native.launch_plan()
        traffic, why = bench.traffic_for(k, plan)
        assert traffic is not None, f"{k}: {why}"
        assert 0.95 < traffic / bench.bytes_min(k, *bench.BENCH[k]) < 1.05
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_gpu_arm_single_kernel_mode_and_tuning_flag():
    """`bench.py --kernel gesummv --tune rowstream=0` on the device: one JSON line, the tunable
    takes effect (two launches per step instead of one)."""
    lines = {}
    for flag in ("rowstream=1", "rowstream=0"):
        proc = subprocess.run([sys.executable, str(REPO / "bench.py"), "--kernel", "gesummv", "--steps", "2",
                               "--warmup", "3", "--no-e2e", "--no-cpu", "--tune", flag],
                              capture_output=True, text=True, timeout=600)
        assert proc.returncode == 0, proc.stderr[-2000:]
        lines[flag] = _line(proc.stdout)
    on, off = lines["rowstream=1"], lines["rowstream=0"]
    assert on["gpu_launches"] == 2 and off["gpu_launches"] == 4
    for d in (on, off):
        assert d["n_gpus"] == 1 and d["roofline"]["kernel"] == "gesummv" and 3000 < d["value"] < 9000
        assert list(d["per_kernel"]) == ["gesummv"]
