#!/bin/bash
# k_cross_tb2: parity tests, one ncu capture at T256 L0, level costs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tblock.py -q -x -p no:cacheprovider > gpurun_out/pytest_tb.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_tb.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cross_tb2 --launch-skip 1 --launch-count 1 \
   -o gpurun_out/tb2_T256 -f python tools/tb_profile.py 256 > gpurun_out/tb2_prof.log 2>&1
ncu -i gpurun_out/tb2_T256.ncu-rep --page details --csv > gpurun_out/tb2_T256_details.csv 2>&1
grep -E '"Duration"|"DRAM Throughput"|Executed Ipc Active|Issue Slots Busy|Warp Cycles Per Issued|Achieved Occupancy|"Registers Per Thread"' gpurun_out/tb2_T256_details.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
SB_TB=1 timeout 300 python tools/level_costs.py T256 1048576:1 > gpurun_out/lc_T256_tb1.txt 2>&1
SB_TB=1 timeout 300 python tools/level_costs.py C2 1048576:1 > gpurun_out/lc_C2_tb1.txt 2>&1
head -8 gpurun_out/lc_T256_tb1.txt gpurun_out/lc_C2_tb1.txt
