#!/bin/bash
# late round-2 profiles: warm-step launch lists (C2, C3) at the final code,
# the mixed-head planner's launch list and one k_ustream capture
mkdir -p gpurun_out/p3
for c in c2 c3; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/p3/launches_$c.csv python tools/profile_step.py --config $c > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/p3/launches_$c.csv > gpurun_out/p3/launches_${c}_summary.txt 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/p3/launches_mixed.csv python tools/mixed_head.py --no-ref > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/p3/launches_mixed.csv > gpurun_out/p3/launches_mixed_summary.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ustream -s 200 -c 1 \
  -o gpurun_out/p3/k_ustream python tools/mixed_head.py --no-ref > /dev/null 2>&1
echo done
