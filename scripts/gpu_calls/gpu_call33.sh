#!/bin/bash
# rows_kernel 2/SM + spill-free; phase probe (self-timed kernel phases) at N=4 and N=2
mkdir -p gpurun_out; rm -f gpurun_out/status33.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_overlap.py -q -x -p no:cacheprovider > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status33.txt
python scripts/local_sweep.py > gpurun_out/local_fused.json 2> gpurun_out/local_fused.err; echo "local rc=$?" >> gpurun_out/status33.txt
python - > gpurun_out/pack_sweep.json 2> gpurun_out/pack_sweep.err <<'PY'
import json, sys, torch
sys.path.insert(0, '.')
import bench
torch.cuda.set_device(0)
sizes = [65536, 1 << 20, 4 << 20, 9437184, 32 << 20, 102015648 // 4 * 4]
t = bench._exchange_times(None, 1, torch.device('cuda', 0), sizes, kind=2, repeats=20)
print(json.dumps({"kernel": "K1 pack (rows_kernel, 2 CTAs/SM)", "sizes": sizes, "us": [round(x * 1e6, 2) for x in t],
                  "hbm_gbs": [round(2 * s / x / 1e9, 1) for s, x in zip(sizes, t)]}))
PY
echo "pack rc=$?" >> gpurun_out/status33.txt
for NG in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2971$NG scripts/phase_probe.py > gpurun_out/phases_n$NG.json 2> gpurun_out/phases_n$NG.err; echo "phases$NG rc=$?" >> gpurun_out/status33.txt
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench1 rc=$?" >> gpurun_out/status33.txt
tail -1 gpurun_out/pytest_k.log
cat gpurun_out/status33.txt
