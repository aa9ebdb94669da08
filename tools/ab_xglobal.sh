#!/bin/bash
# A/B: f32 assign reading the lo plane by TMA (AC_ASG_X_GLOBAL=0) vs the f32 row from global.
mkdir -p gpurun_out
for v in 1 0 1 0; do
  AC_NVCC_FLAGS="-DAC_ASG_X_GLOBAL=$v" python -m paper_2604_18348_b200.build -f > /dev/null 2>&1
  python tools/bench_lloyd.py 2>/dev/null | grep -A3 "token-order, member" | head -3 > gpurun_out/ab_x_$v.txt
  timeout 600 python bench.py --no-cpu-baseline --no-dense --no-e2e > gpurun_out/ab_xb_$v.log 2>&1
  echo "X_GLOBAL=$v: $(tail -1 gpurun_out/ab_xb_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))') | $(head -3 gpurun_out/ab_x_$v.txt | tr '\n' ' ')" >> gpurun_out/ab_x.txt
done
