#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attn_fa4 -c 1 --profile-from-start off -o gpurun_out/attn_fa4 python tools/profile_step.py > gpurun_out/ncu_attn.log 2>&1
