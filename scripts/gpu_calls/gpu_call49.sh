#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status49.txt
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29821 scripts/run_profiles.py --steps 10 --only synth_1000 > gpurun_out/profiles_synth_n4.json 2> gpurun_out/profiles_synth_n4.err; echo "synth rc=$?" >> gpurun_out/status49.txt
cat gpurun_out/status49.txt
