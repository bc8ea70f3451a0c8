#!/bin/bash
mkdir -p gpurun_out

timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tail --launch-skip 2 --launch-count 1 \
   -o gpurun_out/tail_C2 -f python tools/tail_profile.py C2 > gpurun_out/tail_prof.log 2>&1
tail -2 gpurun_out/tail_prof.log
