#!/bin/bash
# bench one workload across library variants: tools/gpu_variants.sh W "name1 name2 ..." (default = in-tree lib)
W=$1; VS=$2
mkdir -p gpurun_out
for V in $VS; do
  if [ "$V" = default ]; then L=""; else L="$PWD/_variants/$V/libsparsh_b200.so"; fi
  SB_LIB=$L timeout 600 python bench.py --steps 5 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/var_${W}_$V.json 2> gpurun_out/var_${W}_$V.err
  python - <<PY
import json
try:
    d = json.load(open("gpurun_out/var_${W}_$V.json"))
except Exception as e:
    print("$W $V", "no line", e, open("gpurun_out/var_${W}_$V.err").read()[-600:]); raise SystemExit
r = d["roofline"]
print("$W $V", f"solve {d['value']*1e3:.2f} ms it {d['config']['iterations']} jac {r['launch_ms']*1e3:.1f} us {r['achieved']:.0f} GB/s ({r['frac']:.3f})")
PY
done
