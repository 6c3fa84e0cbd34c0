#!/usr/bin/env python
"""Does kernel time drift with GPU power/thermal state?  Repeats one kernel for a few
seconds, printing time buckets next to NVML clocks / power / temperature samples."""
import statistics
import sys
import threading
import time
from pathlib import Path

import pynvml
import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from bench import Suite  # noqa: E402
from paper_1205_1098_b200 import _native  # noqa: E402

torch.cuda.set_device(0)
_native.load()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        try:
            samples.append((time.perf_counter(),
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                            pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU),
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        except Exception as exc:  # noqa: BLE001
            samples.append((time.perf_counter(), repr(exc)))
        time.sleep(0.02)


suite = Suite(torch, 0, 1, ("axpydot", "bicgk", "atax", "gesummv", "gemver"))
torch.cuda.synchronize()
time.sleep(3.0)                      # let the GPU idle / cool
th = threading.Thread(target=sampler, daemon=True)
th.start()
for name, secs in (("axpydot", 4.0), ("atax", 4.0), ("bicgk", 4.0)):
    t_end = time.perf_counter() + secs
    rows = []
    while time.perf_counter() < t_end:
        evs = []
        for _ in range(50):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            suite.launch(name)
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        rows.append((time.perf_counter(), statistics.median(a.elapsed_time(b) for a, b in evs)))
    t0 = rows[0][0]
    for t, ms in rows[:: max(1, len(rows) // 12)]:
        near = min((s for s in samples if len(s) > 2), key=lambda s: abs(s[0] - t))
        print(f"{name:8s} t={t - t0:5.2f}s  {ms:.4f} ms   sm={near[1]} MHz mem={near[2]} MHz "
              f"power={near[3]:.0f} W temp={near[4]} C reasons=0x{near[5]:x}", flush=True)
    time.sleep(2.0)
stop.set()
