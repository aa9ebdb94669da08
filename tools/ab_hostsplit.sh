#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
 for sp in 1 2 4; do
  for c in c3 c1; do
    AC_STEADY_SPLIT_HOST=$sp timeout 900 python bench.py --config $c --no-cpu-baseline --no-dense > gpurun_out/b.log 2>&1
    echo "split_host=$sp $c $(tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d[\"ms_per_step\"],3), round(d[\"e2e\"][\"ms_per_step\"],3))")" >> gpurun_out/ab_hs.txt
  done
 done
done
