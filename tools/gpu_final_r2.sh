#!/bin/bash
# end-of-round validation at HEAD: full GPU suite, smoke, C2 bench line, reference arm
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
timeout 1200 python bench.py > gpurun_out/final/bench_c2.log 2>&1; echo "bench rc=$?" >> gpurun_out/final/bench_c2.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/final/bench_ref.log
echo done
