#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_box2.py -q -x -p no:cacheprovider > gpurun_out/pytest_box2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_box2.log
for B in 1 0; do
  SB_BOX2=$B timeout 300 python tools/level_costs.py T256 1048576:1 > gpurun_out/lc_T256_box$B.txt 2>&1
  SB_BOX2=$B timeout 300 python tools/level_costs.py C2 1048576:1 > gpurun_out/lc_C2_box$B.txt 2>&1
done
paste gpurun_out/lc_T256_box1.txt gpurun_out/lc_T256_box0.txt | cut -c1-130
paste gpurun_out/lc_C2_box1.txt gpurun_out/lc_C2_box0.txt | cut -c1-130
