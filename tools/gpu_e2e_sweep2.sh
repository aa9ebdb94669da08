#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/e2e_sweep2.txt
run() { echo "$1 out_chunks=$2 $(AC_STEADY_OUT_CHUNKS=$2 timeout 600 python bench.py --config $1 --no-cpu-baseline --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["e2e"]["ms_per_step"],3))')" >> gpurun_out/e2e_sweep2.txt; }
for oc in 1 2 3; do run c3 $oc; done
for oc in 2 3 5; do run c2 $oc; done
for oc in 2 3 5; do run c4 $oc; done
for oc in 1 2 3 5; do run c1 $oc; done
echo done
