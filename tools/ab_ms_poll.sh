#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/ab_poll.txt
for rep in 1 2; do for v in 0 4 8; do for c in c3 c2; do
  AC_MS_POLL=$v timeout 300 python tools/cold_steps.py $c 2>/dev/null | tail -2 | sed "s/^/poll=$v $c /" >> gpurun_out/ab_poll.txt
done; done; done
