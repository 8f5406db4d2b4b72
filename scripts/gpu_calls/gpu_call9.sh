#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -k autograd > gpurun_out/pytest_autograd.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 scripts/train_bench.py --steps 30 > gpurun_out/train_n4.json 2> gpurun_out/train_n4.err; echo "train4 rc=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
