#!/bin/bash
# update mode x head-block split A/B on the warm step (C2, C4)
mkdir -p gpurun_out
for cfg in c2 c4; do
for ms in "3 0" "2 1" "2 2" "3 1" "2 3"; do
  set -- $ms
  if [ "$2" = "0" ]; then unset AC_STEADY_SPLIT; else export AC_STEADY_SPLIT=$2; fi
  echo "cfg=$cfg mode=$1 split=$2 $(AC_UPDATE_MODE=$1 timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-dense --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')" >> gpurun_out/ms_split.log
done; done
unset AC_STEADY_SPLIT
echo done
