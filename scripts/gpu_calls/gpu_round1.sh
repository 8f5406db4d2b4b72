#!/bin/bash
# first GPU pass: tests, smoke, backward timings, bench
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
nvidia-smi topo -m >> gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 600 python scripts/measure_backward.py gpurun_out/backward_times_b200.json > gpurun_out/measure.log 2>&1; echo "measure rc=$?" >> gpurun_out/status.txt
[ -f gpurun_out/backward_times_b200.json ] && cp gpurun_out/backward_times_b200.json profiles/
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
