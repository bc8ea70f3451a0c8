#!/bin/bash
# round-2 profiles: launch list of the bench command (eager mode: every kernel a
# separate, profiler-visible launch), full capture of the T256 L0 sweep
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 8000 \
   --log-file gpurun_out/r2_launches_bench_T256.csv python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline \
   > gpurun_out/r2_launches_bench.log 2>&1; echo "launch list rc=$?"; tail -2 gpurun_out/r2_launches_bench.log
timeout 900 ncu --nvtx --nvtx-include 'prof/' --set full --import-source on --clock-control none \
   -k regex:k_crosspair --launch-skip 0 --launch-count 1 \
   -o gpurun_out/r2_l0_T256 -f python tools/profile_vcycle.py T256 vcycle > gpurun_out/r2_prof_T256.log 2>&1
tail -2 gpurun_out/r2_prof_T256.log
