#!/bin/bash
mkdir -p gpurun_out
AC_UPDATE_MODE=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ustream -c 1 --profile-from-start off -o gpurun_out/ncu_ustream python tools/profile_step.py --config c3 > gpurun_out/ncu_ustream.log 2>&1
echo done
