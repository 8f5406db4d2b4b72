#!/bin/bash
# multi-GPU pass: every gpu test (incl. multi-process IPC), bench at N=1 and N=$NG
NG=${NG:-2}
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:randomly > gpurun_out/pytest_gpu_multi.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench1 rc=$?" >> gpurun_out/status.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $NG --steps 20 --warmup 5 > gpurun_out/bench_n$NG.json 2> gpurun_out/bench_n$NG.err; echo "bench$NG rc=$?" >> gpurun_out/status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus $NG --steps 10 --warmup 3 > gpurun_out/ref_n$NG.json 2> gpurun_out/ref_n$NG.err; echo "ref$NG rc=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
