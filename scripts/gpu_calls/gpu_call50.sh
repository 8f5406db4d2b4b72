#!/bin/bash
# last full check of the committed state
mkdir -p gpurun_out; rm -f gpurun_out/status50.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status50.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status50.txt
tail -1 gpurun_out/smoke.log; tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/status50.txt
