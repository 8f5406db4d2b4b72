#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status16.txt
for NG in 4 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2957$NG scripts/latency_probe.py > gpurun_out/latency_n$NG.json 2> gpurun_out/latency_n$NG.err; echo "latency$NG rc=$?" >> gpurun_out/status16.txt
done
cat gpurun_out/status16.txt
