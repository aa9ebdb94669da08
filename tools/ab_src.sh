#!/bin/bash
# Same-box A/B of alternative SOURCE files for one unit (e.g. the committed
# version vs the working tree).  usage:
#   [AB_CONFIGS="c2 c3"] tools/ab_src.sh <unit.cu> <src A> <src B> ...
mkdir -p gpurun_out build/csrc
unit=$1; shift
out=gpurun_out/ab_src_${unit%.cu}.txt; : > $out
for src in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --extended-lambda --expt-relaxed-constexpr -Iinclude -Ipaper_2604_18348_b200/csrc $AB_NVCC -c $src \
    -o build/csrc/$unit.o || { echo "build failed: $src" >> $out; continue; }
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2604_18348_b200/libadacluster_sm100.so \
    build/csrc/*.o -lcudart
  for cfg in ${AB_CONFIGS:-c2}; do
    r=$(timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense 2>&1 | tail -1)
    echo "[$src] $cfg $(python -c "import json,sys; d=json.loads(sys.argv[1]); print('step %.3f ms attn %.3f ms frac %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms_per_step'], d['roofline']['frac']))" "$r" 2>&1 | tail -1)" >> $out
  done
done
cat $out
