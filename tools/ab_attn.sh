#!/bin/bash
# A/B compile-time variants of one attention unit on the GPU box.
# usage: [AB_NVCC=...] [AB_TEST=...] [AB_CONFIGS=...] tools/ab_attn.sh <unit.cu> "<flags A>" "<flags B>" ...   (flags may be "")
mkdir -p gpurun_out build/csrc
unit=$1; shift
out=gpurun_out/ab_attn.txt; : > $out
for fl in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --extended-lambda --expt-relaxed-constexpr -Iinclude $AB_NVCC $fl -c paper_2604_18348_b200/csrc/$unit \
    -o build/csrc/$unit.o || { echo "build failed: $fl" >> $out; continue; }
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2604_18348_b200/libadacluster_sm100.so \
    build/csrc/*.o -lcudart
  for cfg in ${AB_CONFIGS:-c2}; do
    r=$(timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dense 2>&1 | tail -1)
    echo "[$fl] $cfg $(python -c "import json,sys; d=json.loads(sys.argv[1]); print('step %.3f ms attn %.3f ms frac %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms_per_step'], d['roofline']['frac']))" "$r" 2>&1 | tail -1)" >> $out
  done
  if [ -n "$AB_TEST" ]; then
    timeout 600 python -m pytest -q -x -m gpu $AB_TEST 2>&1 | tail -1 | sed "s/^/[$fl] tests: /" >> $out
  fi
done
cat $out
