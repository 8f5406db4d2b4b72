# AUTO with LL128: multi-GPU suite, bench at N = 2 / 4, every BASELINE profile at N = 4
set -x
python -m pytest tests/test_gpu_multi.py tests/test_gpu_local_group.py -q -p no:cacheprovider --timeout 1200 > gpurun_out/auto_pytest.log 2>&1; tail -3 gpurun_out/auto_pytest.log
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29554 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 scripts/run_profiles.py --only googlenet_noaux_bs64,resnet50_bs32,vgg16_bs32,bert_base_bs32 > gpurun_out/profiles_n4.json 2> gpurun_out/profiles_n4.err
tail -n 2 gpurun_out/*.err
