# LL128 in rounds (all three phases per round of lines): tests with the default (128-line rounds),
# then A/B of the round size (64 / 128 / 256 / one round = the previous kernel) at N = 4 and 2
set -x
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_local_group.py tests/test_gpu_multi.py -q -p no:cacheprovider -x > gpurun_out/rounds_pytest.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity_large.py -q -p no:cacheprovider -x -k "ll128" > gpurun_out/rounds_parity.log 2>&1
tail -n 1 gpurun_out/rounds_pytest.log gpurun_out/rounds_parity.log
for v in "" _r64 _r256 _rall; do
  MGWFBP_B200_LIB=$PWD/paper_1811_11141_b200/_lib/libmgwfbp_b200$v.so python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2961${#v} scripts/algo_sweep.py --mib 1,2,4,8,16,32,64,128 --algos ll128,ll128_one,push > gpurun_out/rd${v}_n4.json 2> gpurun_out/rd${v}_n4.err
  CUDA_VISIBLE_DEVICES=0,1 MGWFBP_B200_LIB=$PWD/paper_1811_11141_b200/_lib/libmgwfbp_b200$v.so python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2962${#v} scripts/algo_sweep.py --mib 1,2,4,8,16,32,64,128 --algos ll128,ll128_one,push > gpurun_out/rd${v}_n2.json 2> gpurun_out/rd${v}_n2.err
done
grep -h Error gpurun_out/rd*.err | head
