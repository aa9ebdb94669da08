#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/auto_thr.txt
for m in 3 1 3 1; do
  echo "c1 mode=$m $(AC_UPDATE_MODE=$m timeout 600 python bench.py --config c1 --no-cpu-baseline --no-dense --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["cold_step_ms"],2))')" >> gpurun_out/auto_thr.txt
done
for t in 512 2048 8192; do
  echo "c2 small=$t $(AC_USM_SMALL=$t timeout 600 python bench.py --config c2 --no-cpu-baseline --no-dense --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["cold_step_ms"],1))')" >> gpurun_out/auto_thr.txt
  echo "c3 small=$t $(AC_USM_SMALL=$t timeout 600 python bench.py --config c3 --no-cpu-baseline --no-dense --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["cold_step_ms"],1))')" >> gpurun_out/auto_thr.txt
done
echo done
