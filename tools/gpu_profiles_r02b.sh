#!/bin/bash
# Late round-2 profile refresh: attention kernels (warm step), k-means++
# kernels (cold step), warm-step launch lists.
mkdir -p gpurun_out/r02b
P="ncu --set full --import-source on --clock-control none"
timeout 900 $P --profile-from-start off -k regex:'k_attn_fa4$' -c 1 -o gpurun_out/r02b/attn64 python tools/profile_step.py --config c2 > gpurun_out/r02b/attn64.log 2>&1
timeout 900 $P --profile-from-start off -k regex:k_attn_fa4_d128 -c 1 -o gpurun_out/r02b/attn128 python tools/profile_step.py --config c4 > gpurun_out/r02b/attn128.log 2>&1
timeout 900 $P -k regex:k_kpp_dist_v -s 60 -c 1 -o gpurun_out/r02b/kpp_dist python tools/cold_steps.py c2 > gpurun_out/r02b/kpp_dist.log 2>&1
timeout 900 $P -k regex:k_kpp_pick -s 60 -c 1 -o gpurun_out/r02b/kpp_pick python tools/cold_steps.py c2 > gpurun_out/r02b/kpp_pick.log 2>&1
CONFIGS="c2 c3 c4" bash tools/gpu_launches.sh
