# ncu evidence at HEAD (one GPU): K1/K4 at 102 MB, the N=1 step's group kernel, the bench launch list
set -x
nvidia-smi nvlink -gt d -i 0 > gpurun_out/nvlink_gt.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
python scripts/rows_bench.py --reps 2 --warmup 1 > gpurun_out/rows_small.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"rows_kernel|bulk_rows" -c 16 -o gpurun_out/rows_prof \
  python scripts/rows_bench.py --reps 2 --warmup 1 > gpurun_out/rows_ncu.log 2>&1
python scripts/profile_step.py --iters 1 > gpurun_out/step_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"fused_oneshot_kernel" -c 54 -o gpurun_out/step_prof \
  python scripts/profile_step.py --iters 1 > gpurun_out/step_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/step_prof.ncu-rep gpurun_out/ncu_step_summary.json > /dev/null 2>&1
ncu -i gpurun_out/step_prof.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size > gpurun_out/step_launches.csv 2>&1
rm -f gpurun_out/step_prof.ncu-rep
python bench.py --quick --steps 3 --warmup 3 > gpurun_out/quick_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_n1.csv \
  python bench.py --quick --steps 3 --warmup 3 > gpurun_out/quick_ncu.log 2>&1
du -sh gpurun_out; ls -la gpurun_out
