#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/ab_coldq.txt
for rep in 1 2; do for v in 1 0; do
  AC_COLD_Q_INERTIA=$v timeout 300 python tools/cold_steps.py c2 2>/dev/null | tail -3 | sed "s/^/q_inertia=$v /" >> gpurun_out/ab_coldq.txt
done; done
