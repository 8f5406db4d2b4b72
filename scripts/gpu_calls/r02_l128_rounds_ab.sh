# same-box A/B: LL128 before rounds (old) vs rounds of 64 / 128 lines, small and large sizes, N = 4
set -x
for v in _old _r64 ""; do
  MGWFBP_B200_LIB=$PWD/paper_1811_11141_b200/_lib/libmgwfbp_b200$v.so python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2963${#v} scripts/algo_sweep.py --mib 1,2,4,8,16,32,64 --algos ll128 --reps 40 > gpurun_out/ab${v}_n4.json 2> gpurun_out/ab${v}_n4.err
done
for v in _old _r64 ""; do
  MGWFBP_B200_LIB=$PWD/paper_1811_11141_b200/_lib/libmgwfbp_b200$v.so python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2964${#v} scripts/algo_sweep.py --mib 1,2,4,8,16,32,64 --algos ll128 --reps 40 > gpurun_out/ab2${v}_n4.json 2> gpurun_out/ab2${v}_n4.err
done
grep -h Error gpurun_out/ab*.err | head
