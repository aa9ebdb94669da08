#!/bin/bash
# bench lines of the per-layer configs C3-C5 (CPU baseline leg off: it is C2's)
mkdir -p gpurun_out/prof
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/prof/bench_c3.log 2>&1
timeout 1200 python bench.py --config c5 --steps 5 --no-cpu-baseline > gpurun_out/prof/bench_c5.log 2>&1
timeout 1500 python bench.py --config c4 --steps 5 --no-cpu-baseline > gpurun_out/prof/bench_c4.log 2>&1
echo done
