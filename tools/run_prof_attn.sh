#!/bin/bash
# instrumented D=64 attention (build/attn_fa4_prof.cu): per-phase clock64 totals per softmax warp
mkdir -p gpurun_out build/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --extended-lambda \
  --expt-relaxed-constexpr -Iinclude -Ipaper_2604_18348_b200/csrc -c build/attn_fa4_prof.cu -o build/csrc/attn_fa4.cu.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2604_18348_b200/libadacluster_sm100.so build/csrc/*.o -lcudart
timeout 600 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-dense > gpurun_out/prof_attn.log 2>&1
grep PROF gpurun_out/prof_attn.log | tail -40 > gpurun_out/prof_attn_lines.txt
