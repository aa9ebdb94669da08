for cfg in "-DAC_SKIP_IDLE=0" "-DAC_SKIP_MASKED=0"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --extended-lambda --expt-relaxed-constexpr -Iinclude $cfg -c paper_2604_18348_b200/csrc/attn_fa4.cu -o build/csrc/attn_fa4.cu.o && \
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2604_18348_b200/libadacluster_sm100.so build/csrc/*.o -lcudart && \
  echo "$cfg" && python tools/debug/fa4_sparse_dbg.py 2>&1 | grep "bad rows"
done
