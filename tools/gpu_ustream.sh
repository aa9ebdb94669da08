#!/bin/bash
# streamed centroid update: parity of the three update modes, Lloyd-chain A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_assign_tc.py -m gpu -x -q -k "split_chain or lloyd" > gpurun_out/ust_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ust_pytest.log
timeout 300 python tools/bench_lloyd.py --config c3 --heads 12 > gpurun_out/ust_lloyd_c3.log 2>&1
timeout 300 python tools/bench_lloyd.py --config c2 --heads 15 > gpurun_out/ust_lloyd_c2.log 2>&1
for m in 1 2; do
  AC_UPDATE_MODE=$m timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/ust_bench_c3_m$m.log 2>&1
  AC_UPDATE_MODE=$m timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/ust_bench_c2_m$m.log 2>&1
done
echo done
