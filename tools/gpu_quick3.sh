#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_q3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_q3.log
for W in T256 C4 C2 C3; do
timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_q3_$W.json 2>/dev/null; echo "$W $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b_q3_$W.json) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/b_q3_$W.json)"
done
