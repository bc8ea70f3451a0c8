#!/bin/bash
# launch list of one 27-point V-cycle (256^3) + a full ncu capture of its L0 Jacobi sweep (wide row patterns)
WL=${1:-P27_256}
mkdir -p gpurun_out
timeout 900 ncu --nvtx --nvtx-include 'prof/' --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_vcycle_$WL.csv python tools/profile_vcycle.py $WL vcycle > gpurun_out/prof_vc_$WL.log 2>&1
timeout 900 ncu --nvtx --nvtx-include 'prof/' --set full --import-source on --clock-control none \
   -k regex:k_rowpat --launch-skip 0 --launch-count 1 \
   -o gpurun_out/wide_l0_$WL -f python tools/profile_vcycle.py $WL vcycle > gpurun_out/prof_full_$WL.log 2>&1
tail -3 gpurun_out/prof_full_$WL.log
