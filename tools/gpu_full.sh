#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_full.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for T in nccl p2p; do
  timeout 600 python bench.py --dist --transport $T --workload T256 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dist_$T.json 2> gpurun_out/bench_dist_$T.err; echo "dist $T rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_dist_$T.json)"; tail -2 gpurun_out/bench_dist_$T.err
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_T256_final.json 2>gpurun_out/bench_T256_final.err; echo "bench rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_T256_final.json)"
