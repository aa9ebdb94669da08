#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/qfirst.txt
AC_H2D_QFIRST=1 timeout 900 python -m pytest tests/test_steady_graph.py tests/test_stack_gpu.py tests/test_config_parity.py -m gpu -x -q 2>&1 | tail -1 >> gpurun_out/qfirst.txt
for c in c3 c2 c4; do for q in 1 0 1 0; do
  echo "$c qfirst=$q $(AC_H2D_QFIRST=$q timeout 600 python bench.py --config $c --no-cpu-baseline --no-dense 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["e2e"]["ms_per_step"],3))')" >> gpurun_out/qfirst.txt
done; done
echo done
