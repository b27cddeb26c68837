# LeNet conv stage A/B: conv1 on tcgen05 (k_lenet_conv_tc, default) vs the warp-MMA conv (MGFWA_LENET_CONV=mma)
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -k lenet -x -q 2>&1 | tail -n 15
timeout 300 python -m pytest tests/test_gpu_headline_parity.py -k "c3" -x -q 2>&1 | tail -n 5
MGFWA_LENET_CONV=mma timeout 300 python -m pytest tests/test_gpu_parity.py -k lenet -x -q 2>&1 | tail -n 2
timeout 300 python scripts/kernel_times.py --workload c3 --gens 2 --iters 5 > gpurun_out/lenet_ct.json
MGFWA_LENET_CONV=mma timeout 300 python scripts/kernel_times.py --workload c3 --gens 2 --iters 5 > gpurun_out/lenet_mma.json
tail -n 1 gpurun_out/lenet_ct.json gpurun_out/lenet_mma.json
MGFWA_LIB=_variants/ct1/libmgfwa_b200.so timeout 300 python -m pytest tests/test_gpu_parity.py -k lenet -x -q 2>&1 | tail -n 2
MGFWA_LIB=_variants/ct1/libmgfwa_b200.so timeout 300 python scripts/kernel_times.py --workload c3 --gens 2 --iters 5 > gpurun_out/lenet_ct1.json
tail -n 1 gpurun_out/lenet_ct1.json
