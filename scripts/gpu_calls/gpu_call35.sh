#!/bin/bash
# LL area 1 MB per source: explicit-LL vs the rest, engine mode, N=4 and N=2; LL tests
mkdir -p gpurun_out; rm -f gpurun_out/status35.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "every_algorithm or large_multirow or bf16_exchange" > gpurun_out/pytest_ll.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status35.txt
for NG in 4 2; do
GRID_DEFAULTS_ONLY=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2973$NG scripts/grid_sweep.py > gpurun_out/gridll_n$NG.json 2> gpurun_out/gridll_n$NG.err; echo "grid$NG rc=$?" >> gpurun_out/status35.txt
done
tail -1 gpurun_out/pytest_ll.log
cat gpurun_out/status35.txt
