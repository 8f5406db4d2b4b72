#!/bin/bash
# bf16 + replan tests on 4 GPUs, then the single-process ncu evidence (scripts/gpu_calls/gpu_ncu2.sh)
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
tail -15 gpurun_out/pytest_gpu.log
cp gpurun_out/status.txt gpurun_out/status_tests.txt
bash scripts/gpu_calls/gpu_ncu2.sh
cat gpurun_out/status_tests.txt
