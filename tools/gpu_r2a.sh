#!/bin/bash
# round-2 GPU payload: full GPU suite, T256 bench (both arms), level costs, smoke
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt
(nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket") > gpurun_out/host.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_T256.json 2> gpurun_out/bench_T256.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_T256.json; tail -3 gpurun_out/bench_T256.err
timeout 300 python tools/level_costs.py T256 > gpurun_out/level_costs_T256.txt 2>&1
timeout 300 python tools/level_costs.py C2 > gpurun_out/level_costs_C2.txt 2>&1
timeout 1200 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/ref_T256.json 2> gpurun_out/ref_T256.err; echo "ref rc=$?"
cat gpurun_out/ref_T256.json; tail -3 gpurun_out/ref_T256.err
