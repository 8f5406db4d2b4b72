#!/bin/bash
# ncu evidence (1 GPU), each capture only after its own command exited 0 without ncu:
#  1. launch list of the bench (quick) -> share of the step per kernel
#  2. --set full of the bench's N=1 step, the fused group kernel (traffic per launch)
#  3. --set full of the standalone hot kernels (profile_kernels.py)
# Reports are summarised on the box and the big step report deleted (gpurun_out <= 64 MiB).
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python bench.py --steps 3 --warmup 3 --quick > gpurun_out/ncu_bench_plain.json 2> gpurun_out/ncu_bench_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 3 --warmup 3 --quick > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?" >> gpurun_out/status.txt
python scripts/profile_step.py --out gpurun_out/profile_step_groups.json > gpurun_out/profile_step_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:fused_oneshot_kernel<\(int\)1>' -o gpurun_out/prof_step python scripts/profile_step.py --out gpurun_out/profile_step_groups.json > gpurun_out/ncu_step.log 2>&1; echo "step rc=$?" >> gpurun_out/status.txt
python scripts/summarize_step.py gpurun_out/prof_step.ncu-rep gpurun_out/profile_step_groups.json gpurun_out/step_summary.json gpurun_out/roofline_traffic.json > gpurun_out/summarize_step.log 2>&1; echo "sumstep rc=$?" >> gpurun_out/status.txt
ncu -i gpurun_out/prof_step.ncu-rep --page source --csv --kernel-name-base demangled --launch-count 1 > gpurun_out/step_source.csv 2>/dev/null
rm -f gpurun_out/prof_step.ncu-rep
python scripts/profile_kernels.py > gpurun_out/profile_kernels_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:rows_kernel|oneshot|twoshot|fused|b16' -c 24 -o gpurun_out/prof_kernels python scripts/profile_kernels.py > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?" >> gpurun_out/status.txt
python scripts/summarize_ncu.py gpurun_out/launches_n1.csv gpurun_out/prof_kernels.ncu-rep gpurun_out/ncu_summary > gpurun_out/summarize_ncu.log 2>&1; echo "sumncu rc=$?" >> gpurun_out/status.txt
du -sh gpurun_out; ls -la gpurun_out | sort -k5 -n | tail -5
cat gpurun_out/status.txt
