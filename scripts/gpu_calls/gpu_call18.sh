#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status18.txt
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 scripts/train_bench.py --steps 30 --ctas 296,64 --priorities -1 --gates 0 --a-scales 4,16,64 > gpurun_out/train_n4.json 2> gpurun_out/train_n4.err; echo "train4 rc=$?" >> gpurun_out/status18.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench2 rc=$?" >> gpurun_out/status18.txt
cat gpurun_out/status18.txt
