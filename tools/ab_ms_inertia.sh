#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/ab_ms.txt
for rep in 1 2; do for v in 1 0; do for c in c3 c2; do
  AC_MS_INERTIA=$v timeout 300 python tools/cold_steps.py $c 2>/dev/null | tail -2 | sed "s/^/ms_inertia=$v $c /" >> gpurun_out/ab_ms.txt
done; done; done
