# LL with the header check after the fold: correctness (1 GPU + multi) and small-message latency at N = 4
set -x
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_local_group.py tests/test_gpu_multi.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ll_tests.log 2>&1; tail -3 gpurun_out/ll_tests.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 scripts/phase_probe.py > gpurun_out/phases_n4_ll.json 2> gpurun_out/phases_n4_ll.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
tail -n 2 gpurun_out/bench_n4.err gpurun_out/bench_n2.err
