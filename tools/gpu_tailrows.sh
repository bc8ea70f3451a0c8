#!/bin/bash
mkdir -p gpurun_out
for T in 8192 16384 32768; do
  for W in C2 T256; do
    SB_TAIL_ROWS=$T timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bt_$T$W.json 2>/dev/null
    echo "tail=$T $W $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bt_$T$W.json) $(grep -o '"vcycle_ms": [0-9.]*' gpurun_out/bt_$T$W.json)"
  done
done
