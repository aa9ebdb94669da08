#!/bin/bash
# LPT issue order of the attention items: test + A/B on C2/C3/C4
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_item_order.py tests/test_steady_graph.py tests/test_config_parity.py -m gpu -x -q > gpurun_out/ord_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ord_pytest.log
for cfg in c3 c2 c4; do
for o in 1 0 1 0; do
  echo "cfg=$cfg order=$o $(AC_ITEM_ORDER=$o timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-dense --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernel_ms_per_step"])')" >> gpurun_out/ord_ab.log
done; done
echo done
