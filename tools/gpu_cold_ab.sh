#!/bin/bash
# cold-step A/B: HEAD vs the tree in ab_old/ (a git worktree of an older commit)
mkdir -p gpurun_out
for cfg in c2 c3; do
  echo "== HEAD $cfg" >> gpurun_out/cold_ab.log
  timeout 600 python tools/cold_steps.py $cfg >> gpurun_out/cold_ab.log 2>&1
  echo "== OLD $cfg" >> gpurun_out/cold_ab.log
  (cd ab_old && timeout 600 python tools/cold_steps.py $cfg) >> gpurun_out/cold_ab.log 2>&1
done
echo done
