#!/bin/bash
# Round profiling recipe (run under gpurun; results in gpurun_out/prof/).
# One ncu invocation per step, each only after the same command ran clean
# without ncu:
#   bash scripts/profile_round.sh launches [workload]   # ncu launch list of the bench command
#   bash scripts/profile_round.sh cap NAME              # one `ncu --set full` capture of a hot kernel
#     NAME: c2_mlp_fitness | c2_explode_map | c2_guides | c2_rank | c2_select | c2_guide_fitness
#           c3_lenet_conv | c3_lenet_conv_tc | c3_lenet_fc | c5_explode_map | c5_mlp_fitness | c4_explode_map
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
case "${1:-launches}" in
launches)
  W=${2:-c2}
  python bench.py --workload $W --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/launches_dry_$W.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${W}_launches.csv \
    python bench.py --workload $W --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launches_$W.log 2>&1
  ;;
cap)
  # name -> kernel regex, launches to skip (initialize + one generation), workload
  declare -A RE=([c2_mlp_fitness]="k_mlp_fitness 4 c2" [c2_explode_map]="k_explode_map 1 c2"
                 [c2_guides]="k_guides 1 c2" [c2_rank]="k_rank 1 c2" [c2_select]="k_select 1 c2"
                 [c2_guide_fitness]="k_mlp_fitness 5 c2"
                 [c3_lenet_conv]="k_lenet_conv 4 c3" [c3_lenet_conv_tc]="k_lenet_conv_tc 4 c3" [c3_lenet_fc]="k_lenet_fc_tc 4 c3"
                 [c5_explode_map]="k_explode_map 1 c5" [c5_mlp_fitness]="k_mlp_fitness 1 c5"
                 [c4_explode_map]="k_explode_map 1 c4")
  set -- $2 ${RE[$2]}
  python scripts/kernel_times.py --workload $4 --gens 2 --iters 2 > $OUT/dry_$1.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o $OUT/$1 -f \
    python scripts/kernel_times.py --workload $4 --gens 2 --iters 2 > $OUT/ncu_$1.log 2>&1
  ;;
esac
echo done
