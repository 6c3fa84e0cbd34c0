#!/usr/bin/env python
"""Tabulate an ncu --csv launch list: one line per distinct kernel (last launch)."""
import csv, re, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
per = collections.OrderedDict()
for r in rows[1:]:
    per.setdefault(r[ix['ID']], {'name': re.sub(r'\(.*', '', r[ix['Kernel Name']])})[r[ix['Metric Name']]] = r[ix['Metric Value']]
last = collections.OrderedDict()
for it in per.values():
    if any(s in it['name'] for s in sys.argv[2:]) or len(sys.argv) == 2:
        last[it['name']] = it
for name, it in last.items():
    t = float(it['gpu__time_duration.sum']) / 1e3
    rd = float(it.get('dram__bytes_read.sum', 0)) ; wr = float(it.get('dram__bytes_write.sum', 0))
    # ncu prints bytes with unit scaling in some versions; keep raw
    print(f"{name[:60]:60s} {t:9.1f} us grid {it.get('launch__grid_size','?'):>6s} regs {it.get('launch__registers_per_thread','?'):>4s} "
          f"warps {float(it.get('sm__warps_active.avg.pct_of_peak_sustained_active',0)):5.1f}% rd {rd:.4g} wr {wr:.4g}")
