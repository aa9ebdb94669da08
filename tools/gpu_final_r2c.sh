#!/bin/bash
mkdir -p gpurun_out/f3
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/f3/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f3/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f3/smoke.log
timeout 1200 python bench.py > gpurun_out/f3/c2.log 2>&1
for c in c3 c4; do timeout 1500 python bench.py --config $c --breakdown > gpurun_out/f3/$c.log 2>&1; done
echo done
