# wide push grid (>= 112 MiB -> 512 CTAs): parity over IPC at N=2 and N=4, then the default sweep
set -x
python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k wide > gpurun_out/wide_pytest_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k wide > gpurun_out/wide_pytest_n2.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29594 scripts/algo_sweep.py --mib 64,96,128,256,400 --algos push,auto > gpurun_out/wide_n4.json 2> gpurun_out/wide_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29595 scripts/algo_sweep.py --bf16 --mib 64,128,256,400 --algos push,auto > gpurun_out/wide_b16_n4.json 2> gpurun_out/wide_b16_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29596 scripts/algo_sweep.py --mib 64,128,256,400 --algos push,auto > gpurun_out/wide_n2.json 2> gpurun_out/wide_n2.err
tail -n 3 gpurun_out/wide_pytest_*.log
