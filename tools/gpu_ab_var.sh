#!/bin/bash
# A/B of variant builds on bench lines: tools/gpu_ab_var.sh "VAR1 VAR2" "WL1 WL2" (VAR: _variants/NAME or 'base')
mkdir -p gpurun_out
for W in $2; do for i in 1 2; do for V in base $1; do
  if [ $V = base ]; then L=$PWD/paper_2007_00056_b200/_lib/libsparsh_b200.so; else L=$PWD/_variants/$V/libsparsh_b200.so; fi
  SB_LIB=$L timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/abv.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/abv.json'));r=d['roofline'];print('$W $V', round(d['ms_per_step'],2), 'L0', round(r['launch_ms']*1e3,1), round((r.get('launch_ms_warm_back_to_back') or 0)*1e3,1), 'vc', r.get('vcycle_ms'))"
done; done; done
