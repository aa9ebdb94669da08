#!/bin/bash
# Full GPU test suite (incl. the reference-suite conformance run) + smoke.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 ${@} > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
