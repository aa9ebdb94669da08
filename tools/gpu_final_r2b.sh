#!/bin/bash
# final state: GPU suite, smoke, C2 line (driver default), C1 lines
mkdir -p gpurun_out/fin
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fin/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin/smoke.log
timeout 1200 python bench.py > gpurun_out/fin/c2.log 2>&1
for c in c1 c1asis c3; do timeout 1200 python bench.py --config $c --breakdown > gpurun_out/fin/$c.log 2>&1; done
echo done
