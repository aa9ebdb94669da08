#!/bin/bash
# A/B of the exp2 polynomial share in the D = 128 attention kernel
mkdir -p gpurun_out; : > gpurun_out/ab_poly128.txt
for v in 1 2 0 3 1 2; do
  AC_NVCC_FLAGS="-DAC_F128_POLY=$v" python -m paper_2604_18348_b200.build -f > /dev/null 2>&1
  for c in c4 c3; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --no-dense --no-e2e > gpurun_out/ab_p.log 2>&1
    echo "F128_POLY=$v $c: $(tail -1 gpurun_out/ab_p.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["roofline"]["kernel_ms_per_step"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')" >> gpurun_out/ab_poly128.txt
  done
  if [ "$v" = "2" ]; then timeout 600 python -m pytest tests/test_config_parity.py -m gpu -q -x 2>&1 | tail -1 | sed "s/^/F128_POLY=$v tests: /" >> gpurun_out/ab_poly128.txt; fi
done
python -m paper_2604_18348_b200.build -f > /dev/null 2>&1
