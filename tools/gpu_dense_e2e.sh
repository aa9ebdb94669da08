#!/bin/bash
mkdir -p gpurun_out/de
for c in c3 c1 c2 c4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/de/$c.log 2>&1; done
echo done
