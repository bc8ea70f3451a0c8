#!/bin/bash
# solve time vs the cluster-tail threshold (SB_TAIL_ROWS)
mkdir -p gpurun_out
for W in C1 C2 T256; do
  for T in 4096 8192 16384 32768; do
    SB_TAIL_ROWS=$T timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bt.json 2>/dev/null
    echo "tail=$T $W $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bt.json) $(grep -o '"vcycle_ms": [0-9.]*' gpurun_out/bt.json)"
  done
done
