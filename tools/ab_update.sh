mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-dense 2>&1 | tail -1 > gpurun_out/b1.json
python tools/profile_cold.py 2>&1 | head -14 > gpurun_out/cold.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --extended-lambda --expt-relaxed-constexpr -Iinclude --fmad=false -DAC_UPDATE_BULK=0 -c paper_2604_18348_b200/csrc/cluster.cu -o build/csrc/cluster.cu.o && nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2604_18348_b200/libadacluster_sm100.so build/csrc/*.o -lcudart
python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-dense 2>&1 | tail -1 > gpurun_out/b0.json
