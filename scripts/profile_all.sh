#!/bin/bash
# Evidence run (one gpurun call): bench lines of every workload, the
# reference arm, then one ncu full capture per hot kernel (each after its
# dry run), launch lists of C2 and C3.  Output: gpurun_out/prof/.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py --steps 50 --warmup 5 > $OUT/bench_c2.json 2> $OUT/bench.err
: > $OUT/bench_workloads.jsonl
for w in c1 c4 c4a c3 c5 net5 net9; do
  steps=50; [ $w = c3 ] && steps=10; [ $w = c5 ] && steps=4
  timeout 900 python bench.py --workload $w --steps $steps --warmup 3 >> $OUT/bench_workloads.jsonl 2>> $OUT/bench.err
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_c2_reference.json 2>> $OUT/bench.err
python scripts/kernel_times.py --workload c2 > $OUT/kt_c2.json
python scripts/kernel_times.py --workload c3 --gens 2 --iters 5 > $OUT/kt_c3.json
for k in c2_explode_map c2_mlp_fitness c2_guides c2_rank c2_select c2_guide_fitness c3_lenet_conv_tc c3_lenet_fc c4_explode_map c5_explode_map c5_mlp_fitness; do
  timeout 900 bash scripts/profile_round.sh cap $k
done
timeout 900 bash scripts/profile_round.sh launches c2
timeout 900 bash scripts/profile_round.sh launches c3
# summarise on the box (the full reports exceed gpurun's 64 MiB copy-back)
python scripts/ncu_summarize.py report $OUT/c*.ncu-rep $OUT/ncu_full_hot_kernels.json
for k in c2_explode_map c2_mlp_fitness c3_lenet_conv_tc; do
  [ -f $OUT/$k.ncu-rep ] && ncu -i $OUT/$k.ncu-rep --page source --csv --print-source sass > $OUT/${k}_source.csv 2>/dev/null
done
python scripts/ncu_summarize.py launches $OUT/c2_launches.csv $OUT/c2_launches.md 40
python scripts/ncu_summarize.py launches $OUT/c3_launches.csv $OUT/c3_launches.md
rm -f $OUT/*.ncu-rep
echo all done
