#!/bin/bash
# PDL in the large steady steps with the dependents triggered at kernel exit
mkdir -p gpurun_out; : > gpurun_out/ab_pdl_late.txt
for v in 0 1; do
  AC_NVCC_FLAGS="-DAC_PDL_EARLY=$v" python -m paper_2604_18348_b200.build -f > /dev/null 2>&1
  for c in c2 c3; do
    for rows in 0 1000000000; do
      r=$(AC_PDL_STEADY_ROWS=$rows timeout 600 python bench.py --config $c --no-cpu-baseline --no-dense --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))')
      echo "EARLY=$v $c steady_pdl_rows=$rows: $r" >> gpurun_out/ab_pdl_late.txt
    done
  done
done
python -m paper_2604_18348_b200.build -f > /dev/null 2>&1
