#!/bin/bash
# bench lines for C2 (default), C1, C3, C4 + ncu of the L0 sweep
mkdir -p gpurun_out
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for W in C1 C3 C4; do
  timeout 600 python bench.py --steps 5 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
done
timeout 600 ncu --nvtx --nvtx-include "prof/" --set full --import-source on --clock-control none -k regex:k_rowpat -s 0 -c 1 \
   -o gpurun_out/sell_l0 -f python tools/profile_vcycle.py C2 vcycle > gpurun_out/prof_sell.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "prof/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_vcycle_C2.csv python tools/profile_vcycle.py C2 vcycle > gpurun_out/prof_vc.log 2>&1
for W in C1 C2 C3 C4; do python - <<PY
import json
d = json.load(open("gpurun_out/bench_$W.json"))
r = d["roofline"]
print("$W", f"solve {d['value']*1e3:.2f} ms e2e {d['e2e']['value']*1e3:.2f} ms it {d['config']['iterations']} L{d['config']['levels']} "
      f"jac {r['achieved']:.0f} GB/s ({r['frac']:.3f}) csr-eq {r['csr_equiv_gbs']:.0f} vcycle {r['vcycle_ms']:.3f} ms solve {r['solve_gbs']:.0f} GB/s ({r['solve_frac']:.3f}) cpu {d.get('cpu_baseline',{}).get('value')}")
PY
done
