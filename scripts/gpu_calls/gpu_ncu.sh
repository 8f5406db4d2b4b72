#!/bin/bash
# ncu evidence (1 GPU): launch list of the bench step + full capture of the hot kernels
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python bench.py --steps 3 --warmup 3 --quick > gpurun_out/ncu_bench_plain.json 2> gpurun_out/ncu_bench_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rows_kernel|oneshot|twoshot|spin|clock_mark|stamps_reset" --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 3 --warmup 3 --quick > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?" >> gpurun_out/status.txt
python scripts/profile_kernels.py > gpurun_out/profile_kernels_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"rows_kernel|oneshot|twoshot" -c 12 -o gpurun_out/prof_kernels python scripts/profile_kernels.py > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
