#!/bin/bash
# ncu captures of the HBM-bound kernels of a warm C2 step (achieved GB/s)
mkdir -p gpurun_out/prof
for k in k_permute_rows16_heads k_l2norm_v k_envelopes_w k_q_layout_rows k_scatter k_problem_xx_v; do
  timeout 600 ncu --set full --clock-control none -k regex:$k -c 1 --profile-from-start off \
    -o gpurun_out/prof/$k python tools/profile_step.py > /dev/null 2>&1
done
echo done
