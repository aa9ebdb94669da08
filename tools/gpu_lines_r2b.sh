#!/bin/bash
# refresh the per-config bench lines (C2 and the reference arm were refreshed separately)
mkdir -p gpurun_out/lines
for c in c1 c1asis c3 c4 c5; do
  s=$SECONDS
  timeout 1500 python bench.py --config $c --breakdown > gpurun_out/lines/$c.log 2>&1
  echo "$c rc=$? wall=$((SECONDS - s))s" >> gpurun_out/lines/rc.txt
done
echo done
