# 1 GPU: ONE ncu --set full of the 54 launches of the N=1 step's group kernel at HEAD
set -x
python scripts/profile_step.py --iters 1 > gpurun_out/step_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"fused_oneshot_kernel" -c 54 -o gpurun_out/step_prof \
  python scripts/profile_step.py --iters 1 > gpurun_out/step_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/step_prof.ncu-rep gpurun_out/ncu_step_summary.json --sha 8b7f4723cf98 \
  --traffic "fused K1+K4 (N=1)@N1=fused_oneshot_kernel" \
  --note "ncu --set full --clock-control none of the 54 fused_oneshot_kernel<1> launches of one bench N=1 iteration (scripts/profile_step.py) at 8b7f4723cf98; algorithmic bytes 4 x group bytes per launch (gpurun_out/profile_step_groups.json)" > gpurun_out/step_summary.log 2>&1
ncu -i gpurun_out/step_prof.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size > gpurun_out/step_launches.csv 2>&1
cp profiles/roofline_traffic.json gpurun_out/roofline_traffic_step.json
rm -f gpurun_out/step_prof.ncu-rep
du -sh gpurun_out
