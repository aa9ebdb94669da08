#!/bin/bash
# same-box A/B of the member-order update geometry (rows per stage, stages,
# centres per CTA) on C2 / C3 / C4
AB_CONFIGS="c2 c3 c4" bash tools/ab_attn.sh cluster.cu "" "-DAC_UPD_ROWS=16" "-DAC_UPD_WARPS=1" \
  "-DAC_UPD_ROWS=16 -DAC_UPD_WARPS=1" "-DAC_UPD_ROWS=16 -DAC_UPD_STAGES=2" "" > /dev/null 2>&1
cp gpurun_out/ab_attn.txt gpurun_out/ab_update_geom.txt
