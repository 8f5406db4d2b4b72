#!/bin/bash
# programmatic dependent launch of each group's exchange (fill -> exchange)
mkdir -p gpurun_out; rm -f gpurun_out/status39.txt
timeout 900 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/pytest_pdl1.log 2>&1; echo "pytest1 rc=$?" >> gpurun_out/status39.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "emulate or criterion_8 or replan" > gpurun_out/pytest_pdl2.log 2>&1; echo "pytest2 rc=$?" >> gpurun_out/status39.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n1_pdl.json 2> gpurun_out/bench_n1_pdl.err; echo "b1 rc=$?" >> gpurun_out/status39.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pdl > gpurun_out/bench_n1_nopdl.json 2> gpurun_out/bench_n1_nopdl.err; echo "b1n rc=$?" >> gpurun_out/status39.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29761 bench.py --gpus 4 --steps 20 --warmup 5 --no-sweep > gpurun_out/bench_n4_pdl.json 2> gpurun_out/bench_n4_pdl.err; echo "b4 rc=$?" >> gpurun_out/status39.txt
tail -1 gpurun_out/pytest_pdl1.log gpurun_out/pytest_pdl2.log
cat gpurun_out/status39.txt
