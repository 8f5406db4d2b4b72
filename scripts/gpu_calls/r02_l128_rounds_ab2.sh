# same-box A/B after hoisting the per-part ranges into shared memory: old (no rounds) vs rounds of 64 / 128 / 256
set -x
for v in _old _r64 "" _r256; do
  MGWFBP_B200_LIB=$PWD/paper_1811_11141_b200/_lib/libmgwfbp_b200$v.so python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2963${#v} scripts/algo_sweep.py --mib 1,2,4,8,16,32,64,128 --algos ll128,ll128_one --reps 40 > gpurun_out/ac${v}_n4.json 2> gpurun_out/ac${v}_n4.err
  CUDA_VISIBLE_DEVICES=0,1 MGWFBP_B200_LIB=$PWD/paper_1811_11141_b200/_lib/libmgwfbp_b200$v.so python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2964${#v} scripts/algo_sweep.py --mib 1,2,4,8,16,32,64,128 --algos ll128,ll128_one --reps 40 > gpurun_out/ac${v}_n2.json 2> gpurun_out/ac${v}_n2.err
done
grep -h Error gpurun_out/ac*.err | head
