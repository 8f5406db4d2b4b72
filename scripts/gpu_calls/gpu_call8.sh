#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_n4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
for NG in 4 2 1; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2954$NG scripts/train_bench.py --steps 20 > gpurun_out/train_n$NG.json 2> gpurun_out/train_n$NG.err; echo "train$NG rc=$?" >> gpurun_out/status.txt
done
cat gpurun_out/status.txt
