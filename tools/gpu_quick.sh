#!/bin/bash
# quick payload: gpu tests (kernels + cycle + krylov) and the bench line
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
r = d["roofline"]
print(f"solve {d['value']*1e3:.2f} ms  e2e {d['e2e']['value']*1e3:.2f} ms  it {d['config']['iterations']}  "
      f"jacobi {r['achieved']:.0f} GB/s ({r['frac']:.3f}; csr-equiv {r['csr_equiv_gbs']:.0f})  spmv {r['l0_spmv_gbs']:.0f}  vcycle {r['vcycle_ms']:.3f} ms "
      f"({r['vcycle_gbs']:.0f} GB/s)  solve {r['solve_gbs']:.0f} GB/s ({r['solve_frac']:.3f}) clocks {d['clocks']}")
PY
tail -3 gpurun_out/bench.err
