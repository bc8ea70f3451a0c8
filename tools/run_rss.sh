#!/bin/bash
# run a command, print its peak RSS (VmHWM of the process) and wall time
start=$(date +%s.%N)
"$@" &
pid=$!
peak=0
while kill -0 $pid 2>/dev/null; do
  r=$(grep VmHWM /proc/$pid/status 2>/dev/null | awk '{print $2}')
  [ -n "$r" ] && [ "$r" -gt "$peak" ] && peak=$r
  sleep 1
done
wait $pid; rc=$?
end=$(date +%s.%N)
python3 -c "import sys; print(\"peak_rss_gb %.1f wall_s %.1f rc %s\" % (int(sys.argv[1])/1048576, float(sys.argv[3])-float(sys.argv[2]), sys.argv[4]), file=sys.stderr)" $peak $start $end $rc
exit $rc
