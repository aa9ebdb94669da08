#!/bin/bash
# Config-scale parity tests (one/two heads per BASELINE config vs the oracle).
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 2400 python -m pytest tests/test_config_parity.py -m gpu -q -s --durations=0 ${@} > gpurun_out/cfg_parity.log 2>&1
echo "rc=$?" >> gpurun_out/cfg_parity.log
