#!/bin/bash
# A/B of the exp2 polynomial share in the D = 64 attention kernel (current kernel)
mkdir -p gpurun_out; : > gpurun_out/ab_poly64.txt
for v in 1 2 1 2 0 3; do
  AC_NVCC_FLAGS="-DAC_FA4_POLY=$v" python -m paper_2604_18348_b200.build -f > /dev/null 2>&1
  timeout 600 python bench.py --config c2 --no-cpu-baseline --no-dense --no-e2e > gpurun_out/ab_p.log 2>&1
  echo "FA4_POLY=$v c2: $(tail -1 gpurun_out/ab_p.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["roofline"]["kernel_ms_per_step"],3), d["clocks"]["sm_mhz"])')" >> gpurun_out/ab_poly64.txt
done
python -m paper_2604_18348_b200.build -f > /dev/null 2>&1
