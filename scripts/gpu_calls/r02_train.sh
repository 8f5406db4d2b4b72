# real torchvision ResNet-50 training (bs 32/GPU) at N = 4 / 2 with the final kernels: WFBP / MG-WFBP /
# SyncEASGD on the B200 kernels vs DDP (NCCL) vs compute only; plain and interference-aware (--tune)
set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 scripts/train_bench.py --steps 20 --ctas 296,64 --gates 0 > gpurun_out/train_n4.json 2> gpurun_out/train_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 scripts/train_bench.py --steps 20 --tune --ctas 296,64 --gates 0 > gpurun_out/train_n4_tuned.json 2> gpurun_out/train_n4_tuned.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563 scripts/train_bench.py --steps 20 --tune --ctas 296,64 --gates 0 > gpurun_out/train_n2_tuned.json 2> gpurun_out/train_n2_tuned.err
grep -h Error gpurun_out/train*.err | head
