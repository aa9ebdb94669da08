#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_assign_tc.py tests/test_steady_graph.py tests/test_gpu_parity.py tests/test_config_parity.py -m gpu -q -x > gpurun_out/iter_tests.log 2>&1; echo "rc=$?" >> gpurun_out/iter_tests.log
timeout 600 python tools/bench_lloyd.py > gpurun_out/bench_lloyd.log 2>&1
timeout 600 python tools/prof_assign_c2.py >> gpurun_out/bench_lloyd.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-dense > gpurun_out/bench.log 2>&1
