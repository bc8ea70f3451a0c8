#!/bin/bash
# bench lines of every workload on the current build (no CPU baseline)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_full.log
for WL in C1 C2 C3 C4 G128 C5p C5; do
  timeout 900 python bench.py --workload $WL --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_$WL.json 2> gpurun_out/r2_bench_$WL.err
  echo "$WL rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2_bench_$WL.json) $(grep -o '"frac": [0-9.]*' gpurun_out/r2_bench_$WL.json | head -1) $(grep -o '"iterations": [0-9]*' gpurun_out/r2_bench_$WL.json | head -1)"
done
