#!/bin/bash
# A/B: barrier polling with ld.acquire.sys (default) vs relaxed polls + one acquire fence
mkdir -p gpurun_out; rm -f gpurun_out/status34.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29721 scripts/phase_probe.py > gpurun_out/phasesA_n4.json 2> gpurun_out/phasesA_n4.err; echo "A rc=$?" >> gpurun_out/status34.txt
MGWFBP_B200_LIB=$PWD/paper_1811_11141_b200/_lib/variant_relaxpoll.so timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29722 scripts/phase_probe.py > gpurun_out/phasesB_n4.json 2> gpurun_out/phasesB_n4.err; echo "B rc=$?" >> gpurun_out/status34.txt
cat gpurun_out/status34.txt
