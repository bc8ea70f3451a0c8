#!/bin/bash
# launch list (kernel, grid, ncu duration) of one V-cycle: tools/gpu_vclist.sh WL
mkdir -p gpurun_out
WL=${1:-C2}
timeout 600 ncu --nvtx --nvtx-include 'prof/' --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_vc_$WL.csv python tools/profile_vcycle.py $WL vcycle > gpurun_out/prof_vc_$WL.log 2>&1
python tools/launches.py gpurun_out/launches_vc_$WL.csv 1
tail -2 gpurun_out/prof_vc_$WL.log
