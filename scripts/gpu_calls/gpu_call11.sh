#!/bin/bash
# gate + tile changes: GPU suite, real training variants (priority x gate), bench N=1 and N=4
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench1 rc=$?" >> gpurun_out/status.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29543 scripts/train_bench.py --steps 30 --ctas 296,64 --priorities 0,-1 --gates 0,1 > gpurun_out/train_n4.json 2> gpurun_out/train_n4.err; echo "train4 rc=$?" >> gpurun_out/status.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "bench4 rc=$?" >> gpurun_out/status.txt
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/status.txt
