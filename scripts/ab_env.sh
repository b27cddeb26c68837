#!/bin/bash
# A/B of the bench's device-timed ms/generation across environment switches:
#   bash scripts/ab_env.sh "MGFWA_MLP_PRIORITY=0 MGFWA_MLP_PRIORITY=1" "c5"
SETS=${1:-"X=0"}; WLS=${2:-"c2"}
for rep in 1 2; do
for e in $SETS; do
  for w in $WLS; do
    st=30; [ $w = c5 ] && st=3; [ $w = c3 ] && st=5
    env ${e//,/ } timeout 600 python bench.py --workload $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abe.json 2>>gpurun_out/abe.err
    python -c "import json; d=json.load(open('gpurun_out/abe.json')); print('rep$rep $e $w', round(d['ms_per_step'],4), d['value'])"
  done
done
done
