#!/bin/bash
# round profiles: bench line, launch list of one warm step and of the bench
# command, full ncu captures of the three top kernels (summaries as text)
mkdir -p gpurun_out/prof
timeout 1200 python bench.py > gpurun_out/prof/bench.json.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/prof/launches_warm_step.csv python tools/profile_step.py > /dev/null 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 \
  --log-file gpurun_out/prof/launches_bench_cmd.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1
for k in k_attn_fa4 k_assign_tc k_update_w; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 --profile-from-start off \
    -o gpurun_out/prof/$k python tools/profile_step.py > /dev/null 2>&1
done
