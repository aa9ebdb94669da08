#!/bin/bash
mkdir -p gpurun_out
for m in 1 0 1 0; do
  AC_UPDATE_MODE=$m timeout 600 python bench.py --no-cpu-baseline --no-dense --no-e2e --steps 20 > gpurun_out/ab_update_$m.log 2>&1
  echo "mode $m: $(tail -1 gpurun_out/ab_update_$m.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernel_ms_per_step"])')" >> gpurun_out/ab_update.txt
done
