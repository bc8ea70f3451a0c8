#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/pytest_p2p.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_p2p.log
