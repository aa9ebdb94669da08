#!/bin/bash
# streamed centroid update: parity of the three update modes, full-step A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_assign_tc.py -m gpu -x -q -k "split_chain or lloyd" > gpurun_out/ust_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ust_pytest.log
for cfg in c2 c3 c4; do
for m in 1 2 1 2; do
  AC_UPDATE_MODE=$m timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-dense --no-e2e >> gpurun_out/ust_bench_${cfg}_m$m.log 2>&1
done; done
echo done
