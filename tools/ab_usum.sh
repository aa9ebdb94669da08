#!/bin/bash
# A/B: member-order update (mode 1) vs split-chain update with a bounded grid (mode 0).
mkdir -p gpurun_out
for v in "1 2" "0 1" "0 2" "0 4" "1 2" "0 2"; do
  set -- $v
  for c in c2 c3; do
    AC_UPDATE_MODE=$1 AC_USUM_CTAS_PER_SM=$2 timeout 600 python bench.py --config $c --no-cpu-baseline --no-dense --no-e2e > gpurun_out/ab_us.log 2>&1
    echo "mode=$1 cps=$2 $c: $(tail -1 gpurun_out/ab_us.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))')" >> gpurun_out/ab_usum.txt
  done
done
