#!/bin/bash
# ncu launch list (gpu__time_duration per kernel, serialised) of one warm step per config.
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c3}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_$c.csv python tools/profile_step.py --config $c > gpurun_out/ncu_launch_$c.log 2>&1
  python tools/launch_summary.py gpurun_out/launches_$c.csv > gpurun_out/launches_$c.txt 2>&1
done
