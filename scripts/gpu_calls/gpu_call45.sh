#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status45.txt
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29801 scripts/train_bench.py --bf16 --steps 30 --ctas 64 --priorities -1 --gates 0 --tune > gpurun_out/train_bf16_n2.json 2> gpurun_out/train_bf16_n2.err; echo "train2 rc=$?" >> gpurun_out/status45.txt
cat gpurun_out/status45.txt
