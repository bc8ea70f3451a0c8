#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_kernels.py tests/test_gpu_cycle.py -q -x -p no:cacheprovider > gpurun_out/pytest_b27.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_b27.log
timeout 600 python bench.py --workload C5p --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b27.json 2> gpurun_out/b27.err; echo "C5p $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b27.json) $(grep -o '"launch_ms": [0-9.]*' gpurun_out/b27.json) $(grep -o '"frac": [0-9.]*' gpurun_out/b27.json)"
bash tools/gpu_ncu_one.sh P27_256 k_boxpair bp
