#!/bin/bash
NG=${NG:-4}
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_n$NG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 scripts/ar_sweep.py > gpurun_out/sweep_n$NG.json 2> gpurun_out/sweep_n$NG.err; echo "sweep$NG rc=$?" >> gpurun_out/status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 scripts/ar_sweep.py > gpurun_out/sweep_n2.json 2> gpurun_out/sweep_n2.err; echo "sweep2 rc=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
