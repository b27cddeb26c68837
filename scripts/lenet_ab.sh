# LeNet A/B: split conv + tcgen05 fc (default), fused (MGFWA_LENET_FUSED=1), fused conv-only probe
python -m pytest tests/test_gpu_parity.py -k lenet -q 2>&1 | tail -n 2
python -m pytest tests/test_gpu_headline_parity.py -k "c3" -q 2>&1 | tail -n 2
MGFWA_LENET_FUSED=1 python -m pytest tests/test_gpu_parity.py -k lenet -q 2>&1 | tail -n 2
python scripts/kernel_times.py --workload c3 --gens 2 --iters 5 > gpurun_out/lenet_split.json
MGFWA_LENET_FUSED=1 python scripts/kernel_times.py --workload c3 --gens 2 --iters 5 > gpurun_out/lenet_fused.json
MGFWA_LENET_FUSED=1 MGFWA_LIB=_variants/lenet_probe/libmgfwa_b200.so python scripts/kernel_times.py --workload c3 --gens 2 --iters 5 > gpurun_out/lenet_probe.json
tail -n 1 gpurun_out/lenet_*.json
