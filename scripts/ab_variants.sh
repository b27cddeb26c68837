#!/bin/bash
# A/B per-kernel timing of library variants (run under gpurun):
#   bash scripts/ab_variants.sh "default base minb2" "c2 c4" [iters]
# default = the in-tree library; others = _variants/<name>/libmgfwa_b200.so
VARS=${1:-"default"}; WLS=${2:-"c2"}; IT=${3:-10}
mkdir -p gpurun_out
for rep in 1 2; do
for v in $VARS; do
  if [ $v = default ]; then L=""; else L="MGFWA_LIB=_variants/$v/libmgfwa_b200.so"; fi
  for w in $WLS; do
    G=3; [ $w = c5 ] && G=1
    env $L timeout 300 python scripts/kernel_times.py --workload $w --gens $G --iters $IT > gpurun_out/ab_${v}_$w.json 2>>gpurun_out/ab.err
    echo "rep$rep $v $w $(cat gpurun_out/ab_${v}_$w.json)"
  done
done
done
