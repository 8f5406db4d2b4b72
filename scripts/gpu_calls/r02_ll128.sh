# LL128 two-shot: GPU suite on 4 GPUs (LL128 in the local-group, emulated, IPC and stress tests), then sweeps
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/ll128_pytest_n4.log 2>&1
tail -n 5 gpurun_out/ll128_pytest_n4.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29597 scripts/algo_sweep.py --mib 1,2,4,8,16,32,64 --algos push,twoshot,auto,ll128,oneshot,push_oneshot > gpurun_out/l8_n4.json 2> gpurun_out/l8_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29598 scripts/algo_sweep.py --mib 1,2,4,8,16,32,64 --algos push,auto,ll128,push_oneshot > gpurun_out/l8_n2.json 2> gpurun_out/l8_n2.err
tail -n 2 gpurun_out/l8_*.err
