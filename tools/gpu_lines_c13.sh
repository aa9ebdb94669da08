#!/bin/bash
mkdir -p gpurun_out/l2
for c in c1 c1asis c3; do timeout 1200 python bench.py --config $c --breakdown > gpurun_out/l2/$c.log 2>&1; done
echo done
