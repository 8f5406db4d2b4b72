# AUTO with the LL128 one-shot: LL128-related suites, bf16 small-size sweep, bench N = 2 / 4
set -x
timeout 1500 python -m pytest tests/test_gpu_local_group.py tests/test_gpu_multi.py tests/test_host_multiproc.py -q -p no:cacheprovider -x > gpurun_out/l8auto_pytest.log 2>&1
tail -n 3 gpurun_out/l8auto_pytest.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29596 scripts/algo_sweep.py --bf16 --mib 0.0625,0.125,0.25,0.5,1 --algos ll,ll128,ll128_one,auto > gpurun_out/l8one_b16_n4.json 2> gpurun_out/l8one_b16_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29554 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
grep -h Error gpurun_out/*.err | head
