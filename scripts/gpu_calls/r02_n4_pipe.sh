set -x
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_n4b.log 2>&1; tail -3 gpurun_out/pytest_n4b.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 scripts/algo_sweep.py > gpurun_out/sweep_n4.json 2> gpurun_out/sweep_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 scripts/algo_sweep.py > gpurun_out/sweep_n2.json 2> gpurun_out/sweep_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 scripts/nvlink_bytes.py > gpurun_out/nvlink_n4.json 2> gpurun_out/nvlink_n4.err
tail -n 3 gpurun_out/sweep_n4.err gpurun_out/nvlink_n4.err
