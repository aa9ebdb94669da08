#!/bin/bash
# usage: prof_kernel.sh <regex> <name> [count]
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$1 -c ${3:-1} --profile-from-start off -o gpurun_out/$2 python tools/profile_step.py > gpurun_out/ncu_$2.log 2>&1
