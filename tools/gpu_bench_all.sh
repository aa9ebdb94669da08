#!/bin/bash
# Bench lines for every config listed in $CONFIGS.
mkdir -p gpurun_out/lines
for c in ${CONFIGS:-c2 c1 c1asis c3 c4}; do
  s=$SECONDS
  timeout 1500 python bench.py --config $c ${BENCH_ARGS} > gpurun_out/lines/$c.log 2>&1
  echo "$c rc=$? wall=$((SECONDS - s))s" >> gpurun_out/lines/rc.txt
done
