#!/bin/bash
# D=128 tensor-core assign: tests, C2/C3 bench, C3 launch list
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_assign_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2.log
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu_c3.log 2>&1
