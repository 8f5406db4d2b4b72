#!/bin/bash
# re-check of the final committed state on a fresh box
mkdir -p gpurun_out; rm -f gpurun_out/status44.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status44.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status44.txt
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench1 rc=$?" >> gpurun_out/status44.txt
tail -1 gpurun_out/smoke.log; tail -1 gpurun_out/pytest_gpu.log
cat gpurun_out/status44.txt
