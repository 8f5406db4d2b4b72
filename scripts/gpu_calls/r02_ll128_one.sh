# LL128 one-shot: tests touching LL128 (1 GPU + multi-GPU), then small-size sweeps fp32 / bf16 at N = 4 / 2
set -x
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_local_group.py tests/test_gpu_multi.py -q -p no:cacheprovider -x > gpurun_out/l8one_pytest.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_large.py -q -p no:cacheprovider -x -k "ll128" > gpurun_out/l8one_parity.log 2>&1
tail -n 3 gpurun_out/l8one_pytest.log gpurun_out/l8one_parity.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29597 scripts/algo_sweep.py --mib 0.0625,0.125,0.25,0.5,1,2,4 --algos ll,push_oneshot,oneshot,ll128,ll128_one,auto > gpurun_out/l8one_n4.json 2> gpurun_out/l8one_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29596 scripts/algo_sweep.py --bf16 --mib 0.0625,0.125,0.25,0.5,1,2,4 --algos ll,oneshot,ll128,ll128_one,auto > gpurun_out/l8one_b16_n4.json 2> gpurun_out/l8one_b16_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29598 scripts/algo_sweep.py --mib 0.0625,0.125,0.25,0.5,1,2,4 --algos ll,push_oneshot,ll128,ll128_one,auto > gpurun_out/l8one_n2.json 2> gpurun_out/l8one_n2.err
tail -n 2 gpurun_out/l8one_*.err
