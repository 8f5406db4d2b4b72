#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status37.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "large_multirow" > gpurun_out/pytest_ll2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status37.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29751 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "bench4 rc=$?" >> gpurun_out/status37.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29752 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench2 rc=$?" >> gpurun_out/status37.txt
tail -1 gpurun_out/pytest_ll2.log
cat gpurun_out/status37.txt
