#!/bin/bash
# iteration: new row-kernel tests, full GPU suite, C2/C3 bench, warm-step launch list
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_rows_fast.py -x -q > gpurun_out/pytest_rows.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rows.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
grep -q "rc=0" gpurun_out/pytest_gpu.log || exit 1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2.log
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_warm_c2.csv python tools/profile_step.py > /dev/null 2>&1
