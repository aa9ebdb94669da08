#!/bin/bash
# ncu --set full of the key and query tensor-core assignment at C2 (30 heads).
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_assign_tc -c 2 \
  --profile-from-start off -o gpurun_out/asg_c2 python tools/prof_assign_c2.py > gpurun_out/ncu_asg.log 2>&1
python tools/prof_assign_c2.py >> gpurun_out/ncu_asg.log 2>&1
