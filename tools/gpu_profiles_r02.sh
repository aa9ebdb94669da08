#!/bin/bash
# Round-2 profiles: ncu --set full of the top kernels + warm-step launch lists.
mkdir -p gpurun_out/r02
P="ncu --set full --import-source on --clock-control none --profile-from-start off"
timeout 900 $P -k regex:'k_attn_fa4$' -c 1 -o gpurun_out/r02/attn64 python tools/profile_step.py --config c2 > gpurun_out/r02/attn64.log 2>&1
timeout 900 $P -k regex:k_attn_fa4_d128 -c 1 -o gpurun_out/r02/attn128 python tools/profile_step.py --config c4 > gpurun_out/r02/attn128.log 2>&1
timeout 900 $P -k regex:k_assign_tc -c 4 -o gpurun_out/r02/assign python tools/profile_step.py --config c2 > gpurun_out/r02/assign.log 2>&1
timeout 900 $P -k regex:k_update_w -c 2 -o gpurun_out/r02/update python tools/profile_step.py --config c2 > gpurun_out/r02/update.log 2>&1
CONFIGS="c2 c3 c4" bash tools/gpu_launches.sh
