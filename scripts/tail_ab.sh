python -m pytest tests -m gpu -q -x 2>&1 | tail -n 2
for v in default gw2 gw4; do
  if [ $v = default ]; then L=""; else L="MGFWA_LIB=_variants/$v/libmgfwa_b200.so"; fi
  env $L python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/tail_$v.json 2>>gpurun_out/tail.err
  python -c "
import json; d=json.load(open('gpurun_out/tail_$v.json')); kb=d['kernel_breakdown']
print('$v', round(d['ms_per_step'],4), {k: round(x['us'],1) for k,x in kb.items()})"
done
