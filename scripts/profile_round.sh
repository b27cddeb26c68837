#!/bin/bash
# Round profiling recipe (run under gpurun; results in gpurun_out/prof/).
# One ncu invocation per gpurun call, each only after the same command ran
# clean without ncu:
#   bash scripts/profile_round.sh bench      # bench lines for every workload + kernel times
#   bash scripts/profile_round.sh launches   # ncu launch list of the default bench command
#   bash scripts/profile_round.sh cap NAME   # one `ncu --set full` capture of a hot kernel
#     NAME: mlp_fitness | explode_map | guides | rank | lenet_conv | lenet_fc
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
case "${1:-bench}" in
bench)
  python bench.py --steps 50 --warmup 5 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
  : > $OUT/bench_workloads.jsonl
  for w in c1 c4 c3 c5; do
    steps=50; [ $w = c3 ] && steps=10; [ $w = c5 ] && steps=4
    timeout 600 python bench.py --workload $w --steps $steps --warmup 3 >> $OUT/bench_workloads.jsonl 2>> $OUT/bench_workloads.err
  done
  python scripts/kernel_times.py --workload c2 > $OUT/kt_c2.json
  python scripts/kernel_times.py --workload c3 --gens 2 --iters 5 > $OUT/kt_c3.json
  ;;
launches)
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/launches_dry.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/bench_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launches.log 2>&1
  ;;
cap)
  declare -A RE=([mlp_fitness]="k_mlp_fitness 7 c2" [explode_map]="k_explode_map 2 c2" [guides]="k_guides 2 c2"
                 [rank]="k_rank 2 c2" [lenet_conv]="k_lenet_conv 7 c3" [lenet_fc]="k_lenet_fc 7 c3")
  set -- $2 ${RE[$2]}
  python scripts/kernel_times.py --workload $4 --gens 2 --iters 2 > $OUT/dry_$1.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o $OUT/$1 -f \
    python scripts/kernel_times.py --workload $4 --gens 2 --iters 2 > $OUT/ncu_$1.log 2>&1
  ;;
esac
echo done
