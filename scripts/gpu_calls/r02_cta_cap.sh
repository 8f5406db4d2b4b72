# CTA cap for large push two-shot buckets (296 = one resident wave vs 384 / 512)
set -x
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 scripts/algo_sweep.py --mib 32,64,128,256 --algos push,twoshot --max-ctas 296,384,512 > gpurun_out/cap_n4.json 2> gpurun_out/cap_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 scripts/algo_sweep.py --mib 32,64,128,256 --algos push,twoshot --max-ctas 296,384,512 > gpurun_out/cap_n2.json 2> gpurun_out/cap_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29593 scripts/algo_sweep.py --bf16 --mib 32,64,128,256 --algos push --max-ctas 296,384,512 > gpurun_out/cap_b16_n4.json 2> gpurun_out/cap_b16_n4.err
tail -n 2 gpurun_out/cap_*.err
