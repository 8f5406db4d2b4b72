# LL128 at 64 KiB - 32 MiB vs LL / push one-shot / one-shot / AUTO, and LL128 lines per CTA (16..256)
set -x
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29597 scripts/algo_sweep.py --mib 0.0625,0.25,0.5,1,2,4,8,16,32 --algos ll128,auto --per-cta 112,224,896,1792 --per-cta-algos ll128 > gpurun_out/l8s_n4.json 2> gpurun_out/l8s_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29598 scripts/algo_sweep.py --mib 0.0625,0.25,0.5,1,2,4,8,16,32 --algos ll128,auto --per-cta 112,224,896,1792 --per-cta-algos ll128 > gpurun_out/l8s_n2.json 2> gpurun_out/l8s_n2.err
tail -n 2 gpurun_out/l8s_*.err
