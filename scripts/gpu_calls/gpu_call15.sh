#!/bin/bash
# 4 GPUs: multi-rank tests (LL rewrite), latency breakdown, bench N=4 with the full sweep
mkdir -p gpurun_out; rm -f gpurun_out/status15.txt
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status15.txt
for NG in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2955$NG scripts/latency_probe.py > gpurun_out/latency_n$NG.json 2> gpurun_out/latency_n$NG.err; echo "latency$NG rc=$?" >> gpurun_out/status15.txt
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "bench4 rc=$?" >> gpurun_out/status15.txt
tail -3 gpurun_out/pytest_multi.log
cat gpurun_out/status15.txt
