#!/bin/bash
# A/B of two library builds on the T256 bench line: tools/gpu_ab_lib.sh [A.so] [B.so]
mkdir -p gpurun_out
A=${1:-tools/variants/old.so}; B=${2:-paper_2007_00056_b200/_lib/libsparsh_b200.so}
for i in 1 2; do for L in $A $B; do
  SB_LIB=$PWD/$L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab.json'));r=d['roofline'];print('$L', round(d['ms_per_step'],2), round(r['launch_ms']*1e3,1), round(r['launch_ms_warm_back_to_back']*1e3,1), r['vcycle_ms'])"
done; done
