#!/bin/bash
# round-2 final records: bench lines of every workload (T256 with the bounded
# CPU baseline), the reference arm, level costs, launch list and a full ncu
# capture of the T256 L0 sweep (raw pages as CSV)
mkdir -p gpurun_out /tmp/ncu
python bench.py > gpurun_out/r2f_bench_T256.json 2> gpurun_out/r2f_bench_T256.err; echo "T256 rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2f_bench_T256.json)"
for WL in C1 C2 C3 C4 G128 C5p C5; do
  timeout 900 python bench.py --workload $WL --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_$WL.json 2> gpurun_out/r2f_bench_$WL.err
  echo "$WL rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2f_bench_$WL.json) $(grep -o '"frac": [0-9.]*' gpurun_out/r2f_bench_$WL.json | head -1)"
done
for WL in T256 C2; do timeout 600 python tools/level_costs.py $WL 0:1 8192:1 > gpurun_out/r2f_level_costs_$WL.txt 2>&1; done
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -c 7000 \
   --log-file gpurun_out/r2f_launches_bench_T256.csv python bench.py --eager --steps 1 --warmup 0 --no-cpu-baseline \
   > /tmp/ncu/launches.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --nvtx --nvtx-include 'prof/' --set full --import-source on --clock-control none \
   -k regex:k_crosspair --launch-skip 1 --launch-count 1 \
   -o /tmp/ncu/l0 -f python tools/profile_vcycle.py T256 vcycle > /tmp/ncu/l0.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/ncu/l0.ncu-rep --page raw --csv > gpurun_out/r2f_l0_T256_raw.csv
ncu -i /tmp/ncu/l0.ncu-rep --page details --csv > gpurun_out/r2f_l0_T256_details.csv
timeout 1200 python bench.py --impl reference > gpurun_out/r2f_bench_T256_reference_arm.json 2> gpurun_out/r2f_ref.err; echo "ref rc=$? $(head -c 300 gpurun_out/r2f_bench_T256_reference_arm.json)"
