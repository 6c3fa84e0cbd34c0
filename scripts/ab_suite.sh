#!/bin/bash
# Sustained-load A/B of library variants: for each ab_libs/*.so run the suite (100 steps back to
# back: the board reaches its power cap) ROUNDS times, alternating libraries, and print each
# sequence's GB/s.   scripts/ab_suite.sh [rounds] [extra bench.py args]
rounds=${1:-2}; shift
mkdir -p gpurun_out/ab
for r in $(seq 1 $rounds); do
  for so in ab_libs/libbto_b200_*.so; do
    tag=$(basename $so .so | sed 's/libbto_b200_//')
    BTO_B200_LIB=$PWD/$so python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu "$@" > gpurun_out/ab/suite_${tag}_$r.json 2> gpurun_out/ab/suite_${tag}_$r.err
    python - <<PY
import json
d=json.loads(open("gpurun_out/ab/suite_${tag}_$r.json").read().strip().splitlines()[-1])
pk=d["per_kernel"]
print(f"{'$tag':10s} r$r suite {d['value']:7.1f} | " + " ".join(f"{k} {v['gbs']:7.1f} ({v['ms']:.3f}/{v['ms_min']:.3f})" for k,v in pk.items()) + f" | sm {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
  done
done
