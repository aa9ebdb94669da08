#!/bin/bash
# quick GPU iteration: tc assign tests, full gpu suite, bench
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_assign_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --breakdown --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
