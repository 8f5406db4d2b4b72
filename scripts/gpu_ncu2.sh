#!/bin/bash
# ncu evidence (1 GPU), each capture only after its own command exited 0 without ncu:
#  1. launch list of the bench (quick) -> share of the step per kernel
#  2. --set full of the bench's N=1 step, K1 pack launches (traffic per launch)
#  3. --set full of the standalone hot kernels (profile_kernels.py)
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python bench.py --steps 3 --warmup 3 --quick > gpurun_out/ncu_bench_plain.json 2> gpurun_out/ncu_bench_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 3 --warmup 3 --quick > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?" >> gpurun_out/status.txt
python scripts/profile_step.py --out gpurun_out/profile_step_groups.json > gpurun_out/profile_step_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:fused_oneshot_kernel<1>' -o gpurun_out/prof_step python scripts/profile_step.py --out gpurun_out/profile_step_groups.json > gpurun_out/ncu_step.log 2>&1; echo "step rc=$?" >> gpurun_out/status.txt
python scripts/profile_kernels.py > gpurun_out/profile_kernels_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:rows_kernel|oneshot|twoshot|fused' -c 16 -o gpurun_out/prof_kernels python scripts/profile_kernels.py > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
