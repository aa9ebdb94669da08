#!/bin/bash
# full evidence session: tests, smoke, bench (both arms), launch lists, ncu captures
mkdir -p gpurun_out/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/prof/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/prof/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/prof/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/prof/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/prof/smoke.log
timeout 1200 python bench.py > gpurun_out/prof/bench.json.log 2>&1
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/prof/bench_reference.json.log 2>&1
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/prof/bench_c3.json.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/prof/launches_warm_step.csv python tools/profile_step.py > /dev/null 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 \
  --log-file gpurun_out/prof/launches_bench_cmd.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1
for k in k_attn_fa4 k_assign_tc k_update_w k_usum; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 --profile-from-start off \
    -o gpurun_out/prof/$k python tools/profile_step.py > /dev/null 2>&1
done
echo done > gpurun_out/prof/done
