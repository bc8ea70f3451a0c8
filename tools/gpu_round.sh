#!/bin/bash
# One gpurun payload: tests, diag, bench, ncu launch list + full capture of the L0 Jacobi sweep.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 300 python tools/diag_parity.py 2>&1 | tail -12
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
timeout 600 ncu --nvtx --nvtx-include 'prof/' --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_vcycle.csv python tools/profile_vcycle.py C2 vcycle > gpurun_out/prof1.log 2>&1
timeout 600 ncu --nvtx --nvtx-include 'prof/' --set full --import-source on --clock-control none -k regex:k_csr_tile -c 1 \
   -o gpurun_out/jacobi_l0 -f python tools/profile_vcycle.py C2 vcycle > gpurun_out/prof2.log 2>&1
ls -la gpurun_out
