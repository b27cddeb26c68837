# quick C2 / C4 / C5 timing lines (no e2e / cpu baseline) + explode parity
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/q_c2.json 2>gpurun_out/q.err
python bench.py --workload c4 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/q_c4.json 2>>gpurun_out/q.err
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_c5.json 2>>gpurun_out/q.err
for f in gpurun_out/q_*.json; do python -c "
import json; d=json.load(open('$f')); kb=d.get('kernel_breakdown',{})
print('$f', round(d['ms_per_step'],4), {k: round(v['us'],1) for k,v in kb.items() if isinstance(v,dict) and 'us' in v})"; done
