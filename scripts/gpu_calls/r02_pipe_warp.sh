# the per-warp pipelined two-shot: correctness (1 GPU suites) then the sweep at N = 4 and N = 2
set -x
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_local_group.py tests/test_gpu_parity_large.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pipe_tests.log 2>&1; tail -3 gpurun_out/pipe_tests.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 scripts/algo_sweep.py --mib 4,8,16,32,64,128 --algos push,push_pipe,auto --pipe-subs 128,256,1024 > gpurun_out/sweep_pipe_n4.json 2> gpurun_out/sweep_pipe_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 scripts/algo_sweep.py --mib 4,8,16,32,64,128 --algos push,push_pipe,auto --pipe-subs 128,256,1024 > gpurun_out/sweep_pipe_n2.json 2> gpurun_out/sweep_pipe_n2.err
tail -n 2 gpurun_out/sweep_pipe_n4.err gpurun_out/sweep_pipe_n2.err
