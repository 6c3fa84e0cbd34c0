#!/usr/bin/env python
"""Summarise an .ncu-rep (raw page) and a launch-list csv into profiles/ text tables.
    python scripts/ncu_summary.py gpurun_out/prof_r01.ncu-rep gpurun_out/launches.csv profiles/r01/ncu_summary.md
"""
from __future__ import annotations

import csv
import io
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
    ("launch__block_size", "block"), ("launch__cluster_size", "cluster"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem conflicts"),
    ("smsp__inst_executed.sum", "warp insts"),
]


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name).replace("void bto::", "").replace("bto::", "")
    return name.strip()


def main(rep, launches, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = ["# ncu summary (" + rep.split("/")[-1] + ")", "",
             "`ncu --set full --clock-control none --import-source on`, one launch of each hot kernel "
             "inside `bench.py --steps 1 --warmup 3 --no-e2e --no-cpu` (cold-cache, serialised: "
             "compare shares, not absolutes).", ""]
    cols = [(m, label, hdr.index(m)) for m, label in METRICS if m in hdr]
    lines.append("| kernel | " + " | ".join(f"{label} [{units[i]}]" if units[i] else label
                                             for _, label, i in cols) + " |")
    lines.append("|---|" + "---|" * len(cols))
    for r in rows[2:]:
        vals = []
        for m, _, i in cols:
            v = r[i]
            try:
                f = float(v.replace(",", ""))
                v = f"{f:.4g}" if abs(f) < 1e6 else f"{f:.6g}"
            except ValueError:
                pass
            vals.append(v)
        lines.append(f"| `{short(r[hdr.index('Kernel Name')])}` | " + " | ".join(vals) + " |")
    lines += ["", "## launch list (`--metrics gpu__time_duration.sum`, last step)", "",
              "| # | kernel | grid | ms | share of step |", "|---|---|---|---|---|"]
    lrows = [r for r in csv.DictReader(l for l in open(launches) if l.startswith('"'))]
    # the last step: everything from the last vec_kernel (AXPYDOT opens a step) on
    start = max(i for i, r in enumerate(lrows) if 'vec_kernel' in r['Kernel Name'])
    last = lrows[start:]
    total = sum(float(r["Metric Value"].replace(",", "")) for r in last)
    for r in last:
        ns = float(r["Metric Value"].replace(",", ""))
        lines.append(f"| {r['ID']} | `{short(r['Kernel Name'])}` | {r['Grid Size']} | "
                     f"{ns / 1e6:.4f} | {100 * ns / total:.1f}% |")
    lines.append(f"\nstep total under ncu: {total / 1e6:.3f} ms")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
