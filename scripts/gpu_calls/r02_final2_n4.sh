# round-2 final evidence (after LL128) on 4 GPUs: full GPU suite, bench + reference arms at
# N = 1 / 2 / 4, measured Gantt timelines, every BASELINE profile at N = 4, AUTO vs NCCL sweeps
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest_final_n4.log 2>&1; tail -3 gpurun_out/pytest_final_n4.log
CUDA_VISIBLE_DEVICES=0 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_n1.json 2> gpurun_out/ref_n1.err
CUDA_VISIBLE_DEVICES=0 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --impl reference --gpus 2 --steps 20 --warmup 5 > gpurun_out/ref_n2.json 2> gpurun_out/ref_n2.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29553 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/ref_n4.json 2> gpurun_out/ref_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29554 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
python -c "import bench; from paper_1811_11141_b200 import save_profile; save_profile(bench.b200_profile()[0], 'gpurun_out/r50_b200.json')"
python -m paper_1811_11141_b200 emulate --profile gpurun_out/r50_b200.json --nodes 4 --comm-a 1.3e-5 --comm-b 1.9e-12 --iterations 5 --warmup 2 --graph --out gpurun_out/emulate_n4.json --events-csv gpurun_out/timeline_n4_mgwfbp.csv > gpurun_out/emulate_n4.log 2>&1
python -c "import json; json.dump(list(range(2, 55)), open('gpurun_out/sync_plan.json', 'w'))"; python -m paper_1811_11141_b200 emulate --profile gpurun_out/r50_b200.json --nodes 4 --plan gpurun_out/sync_plan.json --iterations 5 --warmup 2 --graph --events-csv gpurun_out/timeline_n4_synceasgd.csv > gpurun_out/emulate_sync_n4.log 2>&1 || true
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 scripts/run_profiles.py --only googlenet_noaux_bs64,resnet50_bs32,vgg16_bs32,bert_base_bs32 > gpurun_out/profiles_n4.json 2> gpurun_out/profiles_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 scripts/algo_sweep.py --mib 0.25,1,2,4,16,32,64,128,256 --algos auto > gpurun_out/auto_n4.json 2> gpurun_out/auto_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29557 scripts/algo_sweep.py --bf16 --mib 0.25,1,4,16,64,128,256 --algos auto > gpurun_out/auto_b16_n4.json 2> gpurun_out/auto_b16_n4.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29558 scripts/algo_sweep.py --mib 0.25,1,2,4,16,32,64,128,256 --algos auto > gpurun_out/auto_n2.json 2> gpurun_out/auto_n2.err
CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29559 scripts/algo_sweep.py --bf16 --mib 0.25,1,4,16,64,128,256 --algos auto > gpurun_out/auto_b16_n2.json 2> gpurun_out/auto_b16_n2.err
grep -h Error gpurun_out/*.err | head
