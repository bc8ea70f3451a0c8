#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_full.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for W in C2 T256; do python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$W', round(d['ms_per_step'],2), d['roofline']['vcycle_ms'], d['gpu_launches'])"; done
