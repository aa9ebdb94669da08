#!/bin/bash
# end-of-session refresh: parity suite, smoke, bench line, reference arm,
# warm-step launch list and the assign-kernel ncu capture
mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/prof/bench.json.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/prof/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/prof/launches_warm_step.csv python tools/profile_step.py > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_assign_tc -c 1 --profile-from-start off \
  -o gpurun_out/prof/k_assign_tc python tools/profile_step.py > /dev/null 2>&1
echo done
