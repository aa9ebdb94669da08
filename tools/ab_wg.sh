#!/bin/bash
# A/B: 3 vs 4 epilogue warpgroups in the tensor-core assignment.
mkdir -p gpurun_out
AC_ASG_WG=4 timeout 900 python -m pytest tests/test_assign_tc.py tests/test_steady_graph.py -m gpu -q -x > gpurun_out/wg4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wg4_tests.log
for w in 3 4 3 4; do
  for c in c2 c3; do
    AC_ASG_WG=$w timeout 600 python bench.py --config $c --no-cpu-baseline --no-dense --no-e2e > gpurun_out/ab_wg_${w}_$c.log 2>&1
    echo "WG=$w $c: $(tail -1 gpurun_out/ab_wg_${w}_$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))')" >> gpurun_out/ab_wg.txt
  done
done
