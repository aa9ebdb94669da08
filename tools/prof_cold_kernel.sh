#!/bin/bash
# ncu capture of one launch of a cold-step kernel (C2 step 0 of a fresh session)
# usage: prof_cold_kernel.sh <regex> <name> [skip]
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$1 -s ${3:-40} -c 1 \
  -o gpurun_out/$2 python tools/cold_steps.py c2 > gpurun_out/ncu_$2.log 2>&1
