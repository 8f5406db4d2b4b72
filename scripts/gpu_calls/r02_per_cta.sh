# push two-shot slots-per-CTA sweep (default rule: 2048-4096) at 2-64 MiB
set -x
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29597 scripts/algo_sweep.py --mib 2,4,8,16,32,64 --algos push --per-cta 256,512,1024,2048,4096 > gpurun_out/per_n4.json 2> gpurun_out/per_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29598 scripts/algo_sweep.py --mib 2,4,8,16,32,64 --algos push --per-cta 256,512,1024,2048,4096 > gpurun_out/per_n2.json 2> gpurun_out/per_n2.err
tail -n 2 gpurun_out/per_*.err
