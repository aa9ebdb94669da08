#!/bin/bash
# steady-step head-block split sweep (AC_STEADY_SPLIT) per config
mkdir -p gpurun_out; out=gpurun_out/split.txt; : > $out
for cfg in ${CFGS:-c2 c3}; do
  for sp in ${SPLITS:-1 2 3 4}; do
    r=$(AC_STEADY_SPLIT=$sp timeout 600 python bench.py --config $cfg --steps 10 --no-cpu-baseline --no-e2e --no-dense 2>&1 | tail -1)
    echo "$cfg split=$sp $(python -c "import json,sys; d=json.loads(sys.argv[1]); print('%.3f ms' % d['ms_per_step'])" "$r" 2>&1 | tail -1)" >> $out
  done
done
cat $out
