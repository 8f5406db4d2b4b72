# bf16 LL128: GPU suite on 4 GPUs, then bf16 sweeps with LL128 at N = 4 / 2
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/b16l8_pytest_n4.log 2>&1
tail -n 5 gpurun_out/b16l8_pytest_n4.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29597 scripts/algo_sweep.py --bf16 --mib 0.25,0.5,1,2,4,8,16,32,64 --algos ll128,auto,push,twoshot > gpurun_out/b16l8_n4.json 2> gpurun_out/b16l8_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29598 scripts/algo_sweep.py --bf16 --mib 0.25,0.5,1,2,4,8,16,32,64 --algos ll128,auto,push > gpurun_out/b16l8_n2.json 2> gpurun_out/b16l8_n2.err
tail -n 2 gpurun_out/b16l8_*.err
