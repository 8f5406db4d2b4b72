# 1 GPU (the driver's shape): full GPU suite, smoke, bench N=1, then ONE ncu: K1/K4 on the 102 MB bucket at HEAD
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_final_1gpu.log 2>&1; tail -3 gpurun_out/pytest_final_1gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1_1gpu.json 2> gpurun_out/bench_n1_1gpu.err
python scripts/rows_bench.py --reps 2 --warmup 1 > gpurun_out/rows_small.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"rows_kernel|bulk_rows" -c 16 -o gpurun_out/rows_prof \
  python scripts/rows_bench.py --reps 2 --warmup 1 > gpurun_out/rows_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/rows_prof.ncu-rep gpurun_out/ncu_rows_summary.json --sha 8b7f4723cf98 \
  --traffic "K1 pack@102MB=bulk_rows_kernel<0>" --traffic "K4 unpack@102MB=bulk_rows_kernel<1>" \
  --note "ncu --set full --clock-control none of scripts/rows_bench.py --reps 2 --warmup 1 at 8b7f4723cf98 (ResNet-50 whole-model bucket, 54 rows, 102,015,648 B): rows_kernel = LDG path, bulk_rows_kernel = TMA bulk path (AUTO); algorithmic bytes 2 x 102,015,648 per launch" > gpurun_out/rows_summary.log 2>&1
cp profiles/roofline_traffic.json gpurun_out/roofline_traffic_rows.json
rm -f gpurun_out/rows_prof.ncu-rep
du -sh gpurun_out
