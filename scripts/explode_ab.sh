# explode variants: kernel times (cold L2) on C2 / C4 / C5-chunked
for v in default sk2 sk3 rk3; do
  if [ $v = default ]; then L=""; else L="MGFWA_LIB=_variants/$v/libmgfwa_b200.so"; fi
  for w in c2 c4; do
    env $L python scripts/kernel_times.py --workload $w --gens 3 --iters 10 > gpurun_out/ex_${v}_$w.json 2>>gpurun_out/ex.err
    echo "$v $w $(cat gpurun_out/ex_${v}_$w.json)"
  done
  env $L python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/exb_$v.json 2>>gpurun_out/ex.err
  python -c "import json; d=json.load(open('gpurun_out/exb_$v.json')); print('$v c2 step', d['ms_per_step'])"
done
MGFWA_LIB=_variants/sk3/libmgfwa_b200.so python -m pytest tests/test_gpu_headline_parity.py tests/test_gpu_parity.py -q -x 2>&1 | tail -n 2
