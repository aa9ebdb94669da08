#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/bench_lloyd.py > gpurun_out/bench_lloyd.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fixup -s 5 -c 1 -o gpurun_out/fix python tools/bench_lloyd.py > gpurun_out/ncu_fix.log 2>&1
