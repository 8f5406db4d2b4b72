#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status20.txt gpurun_out/*.ncu-rep
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29601 scripts/latency_probe.py > gpurun_out/latency_n4.json 2> gpurun_out/latency_n4.err; echo "latency4 rc=$?" >> gpurun_out/status20.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "bench4 rc=$?" >> gpurun_out/status20.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench1 rc=$?" >> gpurun_out/status20.txt
bash scripts/gpu_calls/gpu_ncu2.sh
cat gpurun_out/status20.txt
