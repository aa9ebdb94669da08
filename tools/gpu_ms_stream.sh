#!/bin/bash
# small-batch streamed update in the multi-stage planner: parity + timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_assign_tc.py tests/test_gpu_parity.py tests/test_config_parity.py -m gpu -x -q > gpurun_out/ms_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ms_pytest.log
timeout 300 python tools/mixed_head.py --no-ref > gpurun_out/ms_mixed.log 2>&1
AC_UPDATE_MODE=1 timeout 300 python tools/mixed_head.py --no-ref > gpurun_out/ms_mixed_m1.log 2>&1
for cfg in c1 c2 c3; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-dense --no-e2e > gpurun_out/ms_bench_$cfg.log 2>&1
done
echo done
