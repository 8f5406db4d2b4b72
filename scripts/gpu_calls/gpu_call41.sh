#!/bin/bash
# final round-1 verification: smoke, full GPU suite on 4 GPUs, bench N=1/2/4, reference arms
mkdir -p gpurun_out; rm -f gpurun_out/status41.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status41.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status41.txt
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench1 rc=$?" >> gpurun_out/status41.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29781 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench2 rc=$?" >> gpurun_out/status41.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29782 bench.py --gpus 4 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "bench4 rc=$?" >> gpurun_out/status41.txt
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_n1.json 2> gpurun_out/bench_ref_n1.err; echo "ref1 rc=$?" >> gpurun_out/status41.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29783 bench.py --impl reference --gpus 4 > gpurun_out/bench_ref_n4.json 2> gpurun_out/bench_ref_n4.err; echo "ref4 rc=$?" >> gpurun_out/status41.txt
tail -1 gpurun_out/smoke.log
tail -1 gpurun_out/pytest_gpu.log
cat gpurun_out/status41.txt
