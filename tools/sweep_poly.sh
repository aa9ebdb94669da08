# rebuild the attention unit with variant macros and time the step
rm -f gpurun_out/sweep.txt; mkdir -p gpurun_out
for cfg in "-DAC_FA4_SKIP=0" "-DAC_FA4_SKIP=1"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --extended-lambda --expt-relaxed-constexpr -Iinclude $cfg -c paper_2604_18348_b200/csrc/attn_fa4.cu -o build/csrc/attn_fa4.cu.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2604_18348_b200/libadacluster_sm100.so build/csrc/*.o -lcudart
  echo "$cfg" >> gpurun_out/sweep.txt
  timeout 300 python tools/debug/fa4_sparse_dbg.py 2>&1 | grep "bad rows" >> gpurun_out/sweep.txt
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-dense 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms_per_step'], d['roofline']['frac'])" >> gpurun_out/sweep.txt 2>&1
done
