#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 2500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --dist --steps 3 --warmup 2 > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; tail -c 1500 gpurun_out/bench_dist1.json; tail -5 gpurun_out/bench_dist1.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -c 800 gpurun_out/bench_ref.json
timeout 600 ncu --nvtx --nvtx-include "prof/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_vcycle_C2.csv python tools/profile_vcycle.py C2 vcycle > gpurun_out/prof_vc.log 2>&1
python tools/level_costs.py C2 0:1 1048576:1 2>&1 | grep -v "from L1[0-3]"
