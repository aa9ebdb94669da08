#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/auto_thr2.txt
timeout 900 python -m pytest tests/test_assign_tc.py tests/test_gpu_parity.py tests/test_config_parity.py -m gpu -x -q > gpurun_out/auto_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/auto_pytest.log
for c in c1 c1asis c3 c2; do
  echo "$c $(timeout 600 python bench.py --config $c --no-cpu-baseline --no-dense --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["cold_step_ms"],2))')" >> gpurun_out/auto_thr2.txt
done
echo "mixed $(timeout 300 python tools/mixed_head.py --no-ref 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["gpu_ms"])')" >> gpurun_out/auto_thr2.txt
echo done
