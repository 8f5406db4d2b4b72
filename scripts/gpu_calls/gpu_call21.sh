#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status21.txt
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "absent_peer or dtype_mismatch" > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status21.txt
for NG in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2961$NG scripts/grid_sweep.py > gpurun_out/grid_n$NG.json 2> gpurun_out/grid_n$NG.err; echo "grid$NG rc=$?" >> gpurun_out/status21.txt
done
tail -3 gpurun_out/pytest_new.log
cat gpurun_out/status21.txt
