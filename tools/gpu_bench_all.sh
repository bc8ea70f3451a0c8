#!/bin/bash
# bench lines for every config: C2 (default, with the CPU reference sample), C1,
# C3, C4, the BASELINE target (7-pt Poisson 256^3), the 27-point 256^3 proxy and C5
mkdir -p gpurun_out
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for W in C1 C3 C4 T256 G128; do
  timeout 600 python bench.py --steps 5 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
done
timeout 900 python bench.py --steps 3 --warmup 3 --workload C5p > gpurun_out/bench_C5p.json 2> gpurun_out/bench_C5p.err
[ -z "$NO_C5" ] && timeout 1500 python bench.py --steps 3 --warmup 3 --workload C5 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
for W in C1 C2 C3 C4 T256 G128 C5p C5; do python - <<PY
import json
try:
    d = json.load(open("gpurun_out/bench_$W.json"))
except Exception as e:
    print("$W", "no line", e); raise SystemExit
r = d["roofline"]
print("$W", f"solve {d['value']*1e3:.2f} ms e2e {d['e2e']['value']*1e3:.2f} ms it {d['config']['iterations']} L{d['config']['levels']} "
      f"jac {r['achieved']:.0f} GB/s ({r['frac']:.3f}) traffic {r.get('traffic')} cpu {(d.get('cpu_baseline') or {}).get('value')}")
PY
done
