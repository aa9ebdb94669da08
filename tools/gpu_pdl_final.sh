#!/bin/bash
mkdir -p gpurun_out/pf
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pf/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pf/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/pf/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/pf/smoke.log
for c in c2 c3 c1; do
for o in 1 0; do
  echo "$c pdl=$o $(AC_PDL=$o timeout 600 python bench.py --config $c --no-cpu-baseline --no-dense --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["cold_step_ms"],1))')" >> gpurun_out/pf/ab.txt
done; done
for o in 1 0; do echo "mixed pdl=$o $(AC_PDL=$o timeout 300 python tools/mixed_head.py --no-ref 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["gpu_ms"])')" >> gpurun_out/pf/ab.txt; done
echo done
