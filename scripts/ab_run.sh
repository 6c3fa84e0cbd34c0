#!/bin/bash
# run scripts/sweep.py for each ab_libs/*.so variant (on the GPU box)
kernels=${1:-gemver_pass1}
mkdir -p gpurun_out/ab
for so in ab_libs/libbto_b200_*.so; do
  tag=$(basename $so .so | sed 's/libbto_b200_//')
  BTO_B200_LIB=$PWD/$so python scripts/sweep.py --kernels $kernels --reps 7 --quick --out gpurun_out/ab/$tag.json > gpurun_out/ab/$tag.log 2>&1
  echo "== $tag"; sort -t' ' -k1,1 gpurun_out/ab/$tag.log | awk '{print}' | sort -k1,1 -k10,10nr 2>/dev/null | head -0
  python - <<PY
import json
rows=json.load(open("gpurun_out/ab/$tag.json"))
best={}
for r in rows:
    if r["kernel"] not in best or r["gbs"]>best[r["kernel"]]["gbs"]: best[r["kernel"]]=r
for k,r in best.items():
    cfg={a:b for a,b in r.items() if a not in("kernel","ms_median","ms_min","gbs","frac")}
    print(f"   {k:14s} {r['ms_median']:.4f} ms {r['gbs']:7.1f} GB/s  {cfg}")
PY
done
