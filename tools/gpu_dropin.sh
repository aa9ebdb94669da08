#!/bin/bash
# New drop-in GPU tests + the reference's own suite against the package.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dropin_gpu.py -m gpu -q -x > gpurun_out/dropin.log 2>&1; echo "rc=$?" >> gpurun_out/dropin.log
timeout 1600 python -m pytest tests/test_conformance.py -m gpu -q -s > gpurun_out/conformance.log 2>&1; echo "rc=$?" >> gpurun_out/conformance.log
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_conformance.py > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
