#!/bin/bash
# ncu evidence for every bench line: a full capture (source-level) of the L0
# Jacobi sweep (first k_rowpat launch of one V-cycle) per workload, and the
# launch list of one C2 V-cycle. Summarise here with tools/ncu_summary.py.
mkdir -p gpurun_out
for W in ${@:-C2 C1 C3 C4 T256 P27_256}; do
  timeout 900 ncu --nvtx --nvtx-include 'prof/' --set full --import-source on --clock-control none \
     -k regex:'k_rowpat|k_crosspair|k_boxpair|k_sellg' --launch-skip 0 --launch-count 1 \
     -o gpurun_out/l0_$W -f python tools/profile_vcycle.py $W vcycle > gpurun_out/prof_l0_$W.log 2>&1
  tail -1 gpurun_out/prof_l0_$W.log
done
timeout 600 ncu --nvtx --nvtx-include 'prof/' --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_vcycle_C2.csv python tools/profile_vcycle.py C2 vcycle > gpurun_out/prof_vc.log 2>&1
# summarise on the box (keeps gpurun_out small): raw metric page + json per workload
for W in ${@:-C2 C1 C3 C4 T256 P27_256}; do
  [ -f gpurun_out/l0_$W.ncu-rep ] && python tools/ncu_summary.py gpurun_out/l0_$W.ncu-rep gpurun_out/r1_l0_${W}_raw.csv gpurun_out/ncu_summary_$W.json
  [ "$W" != "C2" ] && rm -f gpurun_out/l0_$W.ncu-rep
done
du -sh gpurun_out
