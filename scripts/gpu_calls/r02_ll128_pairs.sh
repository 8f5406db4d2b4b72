# LL128 with paired lines (120 B payload per 128-B line): LL128 tests, then sweeps vs push / AUTO / NCCL
set -x
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_local_group.py tests/test_gpu_multi.py -q -p no:cacheprovider -x > gpurun_out/pairs_pytest.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_large.py -q -p no:cacheprovider -x -k "ll128" > gpurun_out/pairs_parity.log 2>&1
tail -n 3 gpurun_out/pairs_pytest.log; tail -n 3 gpurun_out/pairs_parity.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29597 scripts/algo_sweep.py --mib 0.25,0.5,1,2,4,8,16,32,64,128 --algos ll128,ll128_one,push,auto > gpurun_out/pairs_n4.json 2> gpurun_out/pairs_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29598 scripts/algo_sweep.py --mib 0.25,0.5,1,2,4,8,16,32,64,128 --algos ll128,ll128_one,push,auto > gpurun_out/pairs_n2.json 2> gpurun_out/pairs_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29596 scripts/algo_sweep.py --bf16 --mib 1,4,16,32,64 --algos ll128,push,auto > gpurun_out/pairs_b16_n4.json 2> gpurun_out/pairs_b16_n4.err
grep -h Error gpurun_out/pairs_*.err | head
