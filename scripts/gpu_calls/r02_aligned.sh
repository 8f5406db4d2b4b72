# 512-B aligned parts / CTA chunks: GPU suite on 4 GPUs, then the slots-per-CTA sweep again
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/aligned_pytest_n4.log 2>&1
tail -n 3 gpurun_out/aligned_pytest_n4.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29597 scripts/algo_sweep.py --mib 2,4,8,16,32,64,96,128 --algos push,twoshot,auto --per-cta 1024,2048,4096 > gpurun_out/al_n4.json 2> gpurun_out/al_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29598 scripts/algo_sweep.py --mib 2,4,8,16,32,64,96,128 --algos push,twoshot,auto --per-cta 1024,2048,4096 > gpurun_out/al_n2.json 2> gpurun_out/al_n2.err
tail -n 2 gpurun_out/al_*.err
