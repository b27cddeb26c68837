for v in default mulptx; do
  if [ $v = default ]; then L=""; else L="MGFWA_LIB=_variants/$v/libmgfwa_b200.so"; fi
  for w in c2 c4; do
    env $L python scripts/kernel_times.py --workload $w --gens 3 --iters 10 > gpurun_out/ex_${v}_$w.json 2>>gpurun_out/ex.err
    echo "$v $w $(cat gpurun_out/ex_${v}_$w.json)"
  done
done
MGFWA_LIB=_variants/mulptx/libmgfwa_b200.so python -m pytest tests/test_gpu_headline_parity.py -k "generation_steps and default" tests/test_gpu_parity.py -q -x 2>&1 | tail -n 2
