#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_configs.py tests/test_gpu_eager.py tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/pytest_q2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_q2.log
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_q2.json 2>/dev/null; echo "T256 $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b_q2.json) $(grep -o '"clocks": {[^}]*}' gpurun_out/b_q2.json)"
done
