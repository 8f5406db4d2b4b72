#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status31.txt
GRID_LARGE=1 GRID_PUSH_ONLY=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 scripts/grid_sweep.py > gpurun_out/gridpush_n4.json 2> gpurun_out/gridpush_n4.err; echo "grid4 rc=$?" >> gpurun_out/status31.txt
cat gpurun_out/status31.txt
