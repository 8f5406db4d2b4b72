#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status29.txt
python scripts/local_sweep.py > gpurun_out/local_default.json 2> gpurun_out/local_default.err; echo "a rc=$?" >> gpurun_out/status29.txt
MGWFBP_B200_LIB=$PWD/paper_1811_11141_b200/_lib/variant_spread2.so python scripts/local_sweep.py > gpurun_out/local_spread2.json 2> gpurun_out/local_spread2.err; echo "b rc=$?" >> gpurun_out/status29.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n1_a.json 2> gpurun_out/bench_n1_a.err; echo "bench_a rc=$?" >> gpurun_out/status29.txt
MGWFBP_B200_LIB=$PWD/paper_1811_11141_b200/_lib/variant_spread2.so timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n1_b.json 2> gpurun_out/bench_n1_b.err; echo "bench_b rc=$?" >> gpurun_out/status29.txt
cat gpurun_out/status29.txt
