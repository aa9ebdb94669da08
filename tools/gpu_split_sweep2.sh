#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/split2.txt
for c in c3 c2 c4; do
for sp in 1 2 3; do
  echo "$c split=$sp $(AC_STEADY_SPLIT=$sp timeout 600 python bench.py --config $c --no-cpu-baseline --no-dense --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))')" >> gpurun_out/split2.txt
done; done
echo done
