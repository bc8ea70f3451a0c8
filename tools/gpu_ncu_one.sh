#!/bin/bash
# full ncu capture (source-level) of the first launch of kernel regex $2 in one V-cycle of workload $1
WL=${1:-P27_256}; K=${2:-k_rowpat}; TAG=${3:-one}
mkdir -p gpurun_out
timeout 900 ncu --nvtx --nvtx-include 'prof/' --set full --import-source on --clock-control none \
   -k regex:$K --launch-skip 0 --launch-count 1 \
   -o gpurun_out/${TAG}_$WL -f python tools/profile_vcycle.py $WL vcycle > gpurun_out/prof_${TAG}_$WL.log 2>&1
tail -2 gpurun_out/prof_${TAG}_$WL.log
