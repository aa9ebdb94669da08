#!/bin/bash
mkdir -p gpurun_out/ck
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ck/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ck/pytest_gpu.log
for c in c1 c3 c2; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/ck/$c.log 2>&1; done
echo done
