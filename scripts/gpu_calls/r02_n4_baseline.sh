set -x
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 900 > gpurun_out/pytest_n4.log 2>&1; tail -3 gpurun_out/pytest_n4.log
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/nvlink_bytes.py > gpurun_out/nvlink_n2.json 2> gpurun_out/nvlink_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 scripts/nvlink_bytes.py > gpurun_out/nvlink_n4.json 2> gpurun_out/nvlink_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 scripts/phase_probe.py > gpurun_out/phases_n4.json 2> gpurun_out/phases_n4.err
tail -2 gpurun_out/nvlink_n2.err gpurun_out/nvlink_n4.err gpurun_out/bench_n4.err gpurun_out/phases_n4.err
