#!/usr/bin/env python
"""profiles/traffic.json from an ncu capture of one bench step.

    python scripts/make_traffic.py gpurun_out/prof_r02.ncu-rep profiles/traffic.json "<source note>"

Reads `ncu -i <rep> --page raw --csv`, walks the launches in order, attributes every kernel
(joins included) to the suite sequence whose main kernel precedes it, and stores per sequence
dram__bytes_read.sum + dram__bytes_write.sum and the kernel instances seen.  bench.py quotes
`roofline.traffic` from this file only while the library still launches these instances
(bench.traffic_for); tests/test_bench_contract.py fails when it does not.
"""
from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys

MAIN = [(r"vec_kernel<2,", "axpydot"), (r"mv_tile_kernel<5,", "bicgk"), (r"atax_cluster_kernel<", "atax"),
        (r"rowstream_kernel<1>", "gesummv"), (r"mv_tile_kernel<3,", "gesummv"),
        (r"mv_tile_kernel<12,", "gemver"), (r"mv_tile_kernel<1,", "gemver")]


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name).replace("bto::", "")
    return name.strip()


def to_bytes(value: str, unit: str) -> float:
    f = float(value.replace(",", ""))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return f * scale.get(unit, 1.0)


def main(rep: str, out: str, note: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    iname, ird, iwr = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    steps: list[dict] = []
    current = None
    for r in rows[2:]:
        name = short(r[iname]).replace(" ", "")
        seq = next((s for pat, s in MAIN if re.search(pat, name)), None)
        if seq == "axpydot" or not steps:
            steps.append({})
        if seq is not None and not (seq == "gemver" and current == "gemver"):
            current = seq
        if current is None:
            continue
        entry = steps[-1].setdefault(current, {"dram_bytes": 0.0, "kernels": [], "all_kernels": []})
        entry["dram_bytes"] += to_bytes(r[ird], units[ird]) + to_bytes(r[iwr], units[iwr])
        label = short(r[iname])
        entry["all_kernels"].append(label)
        if seq is not None:
            entry["kernels"].append(label)
    # the capture window may end inside a step: take the last step that holds all five sequences
    whole = [s for s in steps if len(s) == len({seq for _, seq in MAIN})]
    last = whole[-1] if whole else steps[-1]
    last["_source"] = note
    json.dump(last, open(out, "w"), indent=1)
    for k, v in last.items():
        if k != "_source":
            print(k, f"{v['dram_bytes'] / 1e9:.3f} GB", v["all_kernels"])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "ncu --set full --clock-control none")
