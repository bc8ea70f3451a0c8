#!/bin/bash
# A/B of an env toggle on bench lines: tools/gpu_ab.sh VAR "W1 W2 ..." [tests]
# (runs the GPU tests first when a pytest expression is given as $3)
VAR=$1; WS=$2
mkdir -p gpurun_out
[ -n "$3" ] && timeout 900 python -m pytest tests -m gpu -q -x $3 2>&1 | tail -4
for W in $WS; do for V in 0 1; do
  env $VAR=$V timeout 600 python bench.py --steps 5 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/ab_${W}_$V.json 2> gpurun_out/ab_${W}_$V.err
  python - <<PY
import json
try:
    d = json.load(open("gpurun_out/ab_${W}_$V.json"))
except Exception as e:
    print("$W $VAR=$V", "no line", e, open("gpurun_out/ab_${W}_$V.err").read()[-600:]); raise SystemExit
r = d["roofline"]
print("$W $VAR=$V", f"solve {d['value']*1e3:.2f} ms it {d['config']['iterations']} jac {r['launch_ms']*1e3:.1f} us {r['achieved']:.0f} GB/s ({r['frac']:.3f}) vcycle {r.get('vcycle_ms')}")
PY
done; done
