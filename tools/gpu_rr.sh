#!/bin/bash
mkdir -p gpurun_out
for M in 4611686018427387904 4000000 1000000 0; do
  SB_RR_SPLIT_MIN=$M timeout 300 python tools/level_costs.py T256 1048576:1 > gpurun_out/lc_T256_rr$M.txt 2>&1
  echo "min=$M $(head -4 gpurun_out/lc_T256_rr$M.txt | tail -3 | tr -s ' ' | cut -c1-60 | tr '\n' '|')"
  SB_RR_SPLIT_MIN=$M timeout 300 python tools/level_costs.py C2 1048576:1 > gpurun_out/lc_C2_rr$M.txt 2>&1
  echo "C2 min=$M $(head -3 gpurun_out/lc_C2_rr$M.txt | tail -2 | tr -s ' ' | cut -c1-60 | tr '\n' '|')"
done
