# 1 GPU: ONE ncu pass -- the launch list (gpu__time_duration per launch) of `bench.py --quick` at HEAD
set -x
python bench.py --quick --steps 3 --warmup 3 > gpurun_out/quick_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_n1.csv \
  python bench.py --quick --steps 3 --warmup 3 > gpurun_out/quick_ncu.log 2>&1
du -sh gpurun_out
