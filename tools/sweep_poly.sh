# rebuild the attention unit with variant macros and time the step
for cfg in "-DAC_FA4_POLY=0" "-DAC_FA4_POLY=1" "-DAC_FA4_POLY=2" "-DAC_FA4_POLY=3"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --extended-lambda --expt-relaxed-constexpr -Iinclude $cfg -c paper_2604_18348_b200/csrc/attn_fa4.cu -o build/csrc/attn_fa4.cu.o && \
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2604_18348_b200/libadacluster_sm100.so build/csrc/*.o -lcudart && \
  echo "$cfg" && timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms_per_step'], d['roofline']['frac'])"
done
