#!/bin/bash
# ncu --set full of Jacobi sweeps inside a T256 V-cycle (L0, L1, L2 by launch skip); raw pages as CSV
mkdir -p gpurun_out /tmp/ncu
for SK in 2 7 13; do
timeout 900 ncu --nvtx --nvtx-include 'prof/' -k regex:k_crosspair --launch-skip $SK --launch-count 1 --set full \
  --clock-control none --import-source on -o /tmp/ncu/xp$SK -f python tools/profile_vcycle.py T256 vcycle > /tmp/ncu/xp$SK.log 2>&1
ncu -i /tmp/ncu/xp$SK.ncu-rep --page raw --csv > gpurun_out/xp_T256_skip${SK}_raw.csv
ncu -i /tmp/ncu/xp$SK.ncu-rep --page details --csv > gpurun_out/xp_T256_skip${SK}_details.csv
done
ls -la gpurun_out/xp_T256*
