for cfg in "0 1" "1 1" "1 0"; do set -- $cfg
  MGFWA_PIPELINE=$1 MGFWA_PIPELINE_LC=$2 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pipe_c2_$1$2.json 2>>gpurun_out/pipe.err
  MGFWA_PIPELINE=$1 MGFWA_PIPELINE_LC=$2 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pipe_c5_$1$2.json 2>>gpurun_out/pipe.err
done
python -m pytest tests/test_gpu_headline_parity.py -k "generation_steps and c2" -q 2>&1 | tail -n 2
for f in gpurun_out/pipe_*.json; do echo $f; python -c "import json,sys; d=json.load(open(\"$f\")); print(d[\"ms_per_step\"], d[\"value\"])"; done
tail -5 gpurun_out/pipe.err
