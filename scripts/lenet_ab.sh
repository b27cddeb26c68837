# LeNet fused-kernel A/B: fused (default), conv-only probe, split conv + fc kernels
python -m pytest tests/test_gpu_parity.py -k lenet -q 2>&1 | tail -n 2
python -m pytest tests/test_gpu_headline_parity.py -k "c3" -q 2>&1 | tail -n 2
python scripts/kernel_times.py --workload c3 --gens 2 --iters 5 > gpurun_out/lenet_fused.json
MGFWA_LIB=_variants/lenet_probe/libmgfwa_b200.so python scripts/kernel_times.py --workload c3 --gens 2 --iters 5 > gpurun_out/lenet_probe.json
MGFWA_LENET_FUSED=0 python scripts/kernel_times.py --workload c3 --gens 2 --iters 5 > gpurun_out/lenet_split.json
tail -n 1 gpurun_out/lenet_*.json
