#!/bin/bash
# Final round-2 bench lines for every config + the reference arm (C2) + the
# driver-style launch list of the default bench command.
mkdir -p gpurun_out/lines
for c in c2 c1 c1asis c3 c4 c5; do
  s=$SECONDS
  timeout 1500 python bench.py --config $c --breakdown > gpurun_out/lines/$c.log 2>&1
  echo "$c rc=$? wall=$((SECONDS - s))s" >> gpurun_out/lines/rc.txt
done
s=$SECONDS
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/lines/reference_c2.log 2>&1
echo "reference rc=$? wall=$((SECONDS - s))s" >> gpurun_out/lines/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lines/launches_bench_cmd.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-dense > gpurun_out/lines/ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/lines/launches_bench_cmd.csv > gpurun_out/lines/launches_bench_cmd_summary.txt 2>&1
