#!/bin/bash
# 1 GPU: overlap/kernel tests, bench N=1 (fused N=1 group kernel), ncu evidence
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep
timeout 900 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/pytest_gpu1.log 2>&1; echo "pytest rc=$?" > gpurun_out/status_c13.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench1 rc=$?" >> gpurun_out/status_c13.txt
bash scripts/gpu_calls/gpu_ncu2.sh
tail -2 gpurun_out/pytest_gpu1.log
cat gpurun_out/status_c13.txt
