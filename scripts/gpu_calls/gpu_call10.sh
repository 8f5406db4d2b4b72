#!/bin/bash
# full GPU suite on 4 GPUs + real training with comm-stream priorities + bench N=4
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 scripts/train_bench.py --steps 20 --ctas 296,32 --priorities 0,-1 > gpurun_out/train_n4.json 2> gpurun_out/train_n4.err; echo "train4 rc=$?" >> gpurun_out/status.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "bench4 rc=$?" >> gpurun_out/status.txt
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/status.txt
