#!/bin/bash
mkdir -p gpurun_out
for sp in 1 2 3 2 1 3; do
  for c in c2 c3; do
    AC_STEADY_SPLIT=$sp timeout 600 python bench.py --config $c --no-cpu-baseline --no-dense --no-e2e > gpurun_out/b.log 2>&1
    echo "split=$sp $c $(tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d[\"ms_per_step\"],3))")" >> gpurun_out/ab_split.txt
  done
done
