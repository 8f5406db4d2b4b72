#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status27.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "fused_exchange" > gpurun_out/pytest_push1.log 2>&1; echo "pytest1 rc=$?" >> gpurun_out/status27.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "every_algorithm or large_multirow" > gpurun_out/pytest_push2.log 2>&1; echo "pytest2 rc=$?" >> gpurun_out/status27.txt
for NG in 4 2; do
GRID_DEFAULTS_ONLY=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2967$NG scripts/grid_sweep.py > gpurun_out/gridq_n$NG.json 2> gpurun_out/gridq_n$NG.err; echo "grid$NG rc=$?" >> gpurun_out/status27.txt
done
tail -2 gpurun_out/pytest_push1.log gpurun_out/pytest_push2.log
cat gpurun_out/status27.txt
