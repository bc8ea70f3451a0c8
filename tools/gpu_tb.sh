#!/bin/bash
# fused-sweep (k_cross_tb2) check: parity tests, level costs with/without, T256 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tblock.py tests/test_gpu_eager.py -q -x -p no:cacheprovider > gpurun_out/pytest_tb.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_tb.log
for TB in 1 0; do
  SB_TB=$TB timeout 300 python tools/level_costs.py T256 1048576:1 > gpurun_out/lc_T256_tb$TB.txt 2>&1
  SB_TB=$TB timeout 300 python tools/level_costs.py C2 1048576:1 > gpurun_out/lc_C2_tb$TB.txt 2>&1
done
head -20 gpurun_out/lc_T256_tb1.txt gpurun_out/lc_C2_tb1.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_T256_tb.json 2> gpurun_out/bench_T256_tb.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_T256_tb.json")); r = d["roofline"]
print(f"T256 solve {d['value']*1e3:.2f} ms e2e {d['e2e']['value']*1e3:.2f} it {d['run']['iterations']} vcycle {r['vcycle_ms']*1e3:.0f} us solve_frac {r['solve_frac']:.3f} clocks {d['clocks']}")
PY
tail -3 gpurun_out/bench_T256_tb.err
