#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/splith.txt
for c in c2 c4; do for sh in 2 4 6; do
  echo "$c split_host=$sh $(AC_STEADY_SPLIT_HOST=$sh timeout 600 python bench.py --config $c --no-cpu-baseline --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["e2e"]["ms_per_step"],3))')" >> gpurun_out/splith.txt
done; done
for sh in 1 2 3; do
  echo "c3 split_host=$sh $(AC_STEADY_SPLIT_HOST=$sh timeout 600 python bench.py --config c3 --no-cpu-baseline --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["e2e"]["ms_per_step"],3))')" >> gpurun_out/splith.txt
done
echo done
