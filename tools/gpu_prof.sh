#!/bin/bash
# gpu tests of the cycle + launch lists of one V-cycle for several tail thresholds
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cycle.py tests/test_gpu_kernels.py -q -x 2>&1 | tail -5
for T in 0 1048576; do
  SB_TAIL_ROWS=$T timeout 600 ncu --nvtx --nvtx-include 'prof/' --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches_vc_tail$T.csv python tools/profile_vcycle.py C2 vcycle > gpurun_out/prof_t$T.log 2>&1
done
for T in 0 1048576; do SB_TAIL_ROWS=$T python tools/profile_vcycle.py C2 solve | tail -1; done
