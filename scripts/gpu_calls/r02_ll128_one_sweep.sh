# LL128 one-shot vs LL / push one-shot / one-shot / LL128 two-shot (LL only to its 1 MiB ceiling)
set -x
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29597 scripts/algo_sweep.py --mib 0.0625,0.125,0.25,0.5,1 --algos ll,push_oneshot,oneshot,ll128,ll128_one,auto > gpurun_out/l8one_n4.json 2> gpurun_out/l8one_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29595 scripts/algo_sweep.py --mib 2,4,8 --algos ll128,ll128_one,auto > gpurun_out/l8one_big_n4.json 2> gpurun_out/l8one_big_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29596 scripts/algo_sweep.py --bf16 --mib 0.0625,0.125,0.25,0.5,1,2 --algos ll,ll128,ll128_one,auto > gpurun_out/l8one_b16_n4.json 2> gpurun_out/l8one_b16_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29598 scripts/algo_sweep.py --mib 0.0625,0.125,0.25,0.5,1 --algos ll,push_oneshot,ll128,ll128_one,auto > gpurun_out/l8one_n2.json 2> gpurun_out/l8one_n2.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29594 scripts/algo_sweep.py --mib 2,4,8 --algos ll128,ll128_one,auto > gpurun_out/l8one_big_n2.json 2> gpurun_out/l8one_big_n2.err
grep -h Error gpurun_out/l8one_*.err | head
