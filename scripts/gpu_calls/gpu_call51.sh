#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status51.txt
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "stress or large_multirow or criterion_7" > gpurun_out/pytest_cap.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status51.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29831 bench.py --gpus 2 --no-sweep > gpurun_out/bench_n2_cap.json 2> gpurun_out/bench_n2_cap.err; echo "bench2 rc=$?" >> gpurun_out/status51.txt
tail -n1 gpurun_out/pytest_cap.log
cat gpurun_out/status51.txt
