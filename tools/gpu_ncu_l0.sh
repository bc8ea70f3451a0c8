#!/bin/bash
# launch list of one C2 V-cycle + a full ncu capture (source-level) of the L0 Jacobi sweep
mkdir -p gpurun_out
timeout 600 ncu --nvtx --nvtx-include 'prof/' --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_vcycle_C2.csv python tools/profile_vcycle.py C2 vcycle > gpurun_out/prof_vc.log 2>&1
timeout 900 ncu --nvtx --nvtx-include 'prof/' --set full --import-source on --clock-control none \
   -k regex:k_rowpat --launch-skip 0 --launch-count 1 \
   -o gpurun_out/sell_l0 -f python tools/profile_vcycle.py C2 vcycle > gpurun_out/prof_full.log 2>&1
tail -3 gpurun_out/prof_full.log
ls -la gpurun_out
