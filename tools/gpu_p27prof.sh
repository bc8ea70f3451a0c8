#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hybrid.py tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "residency or C4" > gpurun_out/pytest_fix.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_fix.log
bash tools/gpu_ncu_one.sh P27_256 k_boxpair bp
