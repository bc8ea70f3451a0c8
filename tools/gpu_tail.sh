#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cycle.py tests/test_gpu_krylov.py tests/test_gpu_general.py -q -x -p no:cacheprovider > gpurun_out/pytest_tail.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_tail.log
LC_TRACE=1 timeout 300 python tools/level_costs.py C2 1048576:1 > gpurun_out/lc_C2_tail.txt 2>&1
timeout 300 python tools/level_costs.py T256 1048576:1 > gpurun_out/lc_T256_tail.txt 2>&1
cat gpurun_out/lc_C2_tail.txt; head -4 gpurun_out/lc_T256_tail.txt; grep "L10" gpurun_out/lc_T256_tail.txt
