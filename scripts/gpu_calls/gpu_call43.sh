#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status43.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "fused_exchange" > gpurun_out/pytest_p1.log 2>&1; echo "pytest1 rc=$?" >> gpurun_out/status43.txt
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "every_algorithm or stress or large_multirow" > gpurun_out/pytest_p2.log 2>&1; echo "pytest2 rc=$?" >> gpurun_out/status43.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29791 scripts/phase_probe.py > gpurun_out/phases_n4.json 2> gpurun_out/phases_n4.err; echo "phases4 rc=$?" >> gpurun_out/status43.txt
tail -n1 gpurun_out/pytest_p1.log; tail -n1 gpurun_out/pytest_p2.log
cat gpurun_out/status43.txt
