#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cycle.py tests/test_gpu_krylov.py -q -x -p no:cacheprovider > gpurun_out/pytest_split.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_split.log
for S in 1 0; do
  SB_PROLONG_SPLIT=$S timeout 300 python tools/level_costs.py T256 1048576:1 > gpurun_out/lc_T256_split$S.txt 2>&1
  SB_PROLONG_SPLIT=$S timeout 300 python tools/level_costs.py C2 1048576:1 > gpurun_out/lc_C2_split$S.txt 2>&1
  SB_PROLONG_SPLIT=$S timeout 300 python tools/level_costs.py C1 1048576:1 > gpurun_out/lc_C1_split$S.txt 2>&1
done
paste gpurun_out/lc_T256_split1.txt gpurun_out/lc_T256_split0.txt | head -7 | cut -c1-130
paste gpurun_out/lc_C2_split1.txt gpurun_out/lc_C2_split0.txt | head -5 | cut -c1-130
paste gpurun_out/lc_C1_split1.txt gpurun_out/lc_C1_split0.txt | head -5 | cut -c1-130
for S in 1 0; do
  SB_PROLONG_SPLIT=$S timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_split$S.json 2>/dev/null; echo "T256 split=$S $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b_split$S.json)"
  SB_PROLONG_SPLIT=$S timeout 600 python bench.py --workload C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b2_split$S.json 2>/dev/null; echo "C2 split=$S $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b2_split$S.json)"
done
