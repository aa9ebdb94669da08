mkdir -p gpurun_out build/csrc; out=gpurun_out/ab2.txt; : > $out
for fl in -DAC_ASG_X_GLOBAL=0 -DAC_ASG_X_GLOBAL=1 -DAC_ASG_X_GLOBAL=0 -DAC_ASG_X_GLOBAL=1; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --extended-lambda --expt-relaxed-constexpr -Iinclude --fmad=false $fl -c paper_2604_18348_b200/csrc/assign_tc.cu -o build/csrc/assign_tc.cu.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2604_18348_b200/libadacluster_sm100.so build/csrc/*.o -lcudart
  r=$(timeout 600 python bench.py --no-cpu-baseline --no-dense 2>&1 | tail -1)
  echo "$fl $(python -c "import json,sys; d=json.loads(sys.argv[1]); print('step %.3f e2e %.3f' % (d['ms_per_step'], d['e2e']['ms_per_step']))" "$r")" >> $out
done
cat $out
