#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/pytest_dist.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_dist.log
for WL in C2 T256; do
  timeout 600 python bench.py --dist --workload $WL --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dist_$WL.json 2> gpurun_out/bench_dist_$WL.err; echo "dist $WL rc=$?"
  tail -c 600 gpurun_out/bench_dist_$WL.json; tail -3 gpurun_out/bench_dist_$WL.err
done
