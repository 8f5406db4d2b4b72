# bf16 push two-shot: correctness on one GPU, then bf16 sweeps vs NCCL bf16 at N = 4 and N = 2
set -x
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_local_group.py tests/test_gpu_parity_large.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b16push_tests.log 2>&1; tail -3 gpurun_out/b16push_tests.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 scripts/algo_sweep.py --bf16 --mib 1,4,8,16,32,64,128 --algos twoshot,push,auto > gpurun_out/sweep_b16_n4.json 2> gpurun_out/sweep_b16_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 scripts/algo_sweep.py --bf16 --mib 1,4,8,16,32,64,128 --algos twoshot,push,auto > gpurun_out/sweep_b16_n2.json 2> gpurun_out/sweep_b16_n2.err
python -m pytest tests/test_gpu_multi.py -m gpu -q -x -p no:cacheprovider -k "bf16" > gpurun_out/b16push_multi.log 2>&1; tail -3 gpurun_out/b16push_multi.log
tail -n 2 gpurun_out/sweep_b16_n4.err gpurun_out/sweep_b16_n2.err
