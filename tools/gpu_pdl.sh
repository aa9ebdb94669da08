#!/bin/bash
# selective programmatic dependent launch: parity + A/B (AC_PDL_STEADY_ROWS / AC_PDL_PLANNER)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pdl_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pdl_pytest.log
for cfg in c1 c3 c2; do
for o in 1 0 1 0; do
  echo "cfg=$cfg pdl=$o $(AC_PDL_PLANNER=$o AC_PDL_STEADY_ROWS=$((o*200000)) timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-dense --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["cold_step_ms"])')" >> gpurun_out/pdl_ab.log
done; done
for cfg in c2 c3; do
for o in 1 0; do echo "cold $cfg pdl=$o" >> gpurun_out/pdl_ab.log; AC_PDL_PLANNER=$o timeout 600 python tools/cold_steps.py $cfg 2>&1 | tail -4 >> gpurun_out/pdl_ab.log; done; done
AC_PDL_PLANNER=1 timeout 300 python tools/mixed_head.py --no-ref > gpurun_out/pdl_mixed1.log 2>&1
AC_PDL_PLANNER=0 timeout 300 python tools/mixed_head.py --no-ref > gpurun_out/pdl_mixed0.log 2>&1
echo done
