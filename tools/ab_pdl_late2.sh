#!/bin/bash
# PDL trigger placement on the small chains (C1 steady, mixed-head planner)
mkdir -p gpurun_out; : > gpurun_out/ab_pdl_late2.txt
for v in 0 1; do
  AC_NVCC_FLAGS="-DAC_PDL_EARLY=$v" python -m paper_2604_18348_b200.build -f > /dev/null 2>&1
  for on in 1 0 1 0; do
    r=$(AC_PDL_STEADY_ROWS=$((on*200000)) AC_PDL_PLANNER=$on timeout 600 python bench.py --config c1 --no-cpu-baseline --no-dense --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4))')
    m=$(AC_PDL_PLANNER=$on timeout 300 python tools/mixed_head.py --no-ref 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(min(d["gpu_ms"]),1))')
    echo "EARLY=$v pdl=$on c1 $r mixed $m" >> gpurun_out/ab_pdl_late2.txt
  done
done
python -m paper_2604_18348_b200.build -f > /dev/null 2>&1
