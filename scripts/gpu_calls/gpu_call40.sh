#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status40.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29771 scripts/nvls_tune.py > gpurun_out/nvls_tune_n4.json 2> gpurun_out/nvls_tune_n4.err; echo "nvls4 rc=$?" >> gpurun_out/status40.txt
cat gpurun_out/status40.txt
