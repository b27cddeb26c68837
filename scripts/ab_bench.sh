#!/bin/bash
# A/B of the bench's device-timed ms/generation across library variants:
#   bash scripts/ab_bench.sh "default nopf" "c2 c5"
VARS=${1:-"default"}; WLS=${2:-"c2"}
for rep in 1 2; do
for v in $VARS; do
  if [ $v = default ]; then L=""; else L="MGFWA_LIB=_variants/$v/libmgfwa_b200.so"; fi
  for w in $WLS; do
    st=30; [ $w = c5 ] && st=3; [ $w = c3 ] && st=5
    env $L timeout 600 python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abb_${v}_$w.json 2>>gpurun_out/abb.err
    python -c "import json; d=json.load(open('gpurun_out/abb_${v}_$w.json')); print('rep$rep $v $w', round(d['ms_per_step'],4), d['value'])"
  done
done
done
