#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/e2e_sweep.txt
for c in c3; do
for sh in 1 2 3 4; do for oc in 3 5 8; do
  echo "$c split_host=$sh out_chunks=$oc $(AC_STEADY_SPLIT_HOST=$sh AC_STEADY_OUT_CHUNKS=$oc timeout 600 python bench.py --config $c --no-cpu-baseline --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["e2e"]["ms_per_step"],3))')" >> gpurun_out/e2e_sweep.txt
done; done; done
echo done
