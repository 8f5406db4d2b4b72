# A/B: LL128 poll back-off (0 / 64 / 256 ns between re-polls) at N = 4, LL128 and AUTO
set -x
for v in "" _bo64 _bo256; do
  MGWFBP_B200_LIB=$PWD/paper_1811_11141_b200/_lib/libmgwfbp_b200$v.so python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2960${#v} scripts/algo_sweep.py --mib 1,4,16,32,64,128 --algos ll128,ll128_one,push > gpurun_out/bo${v}_n4.json 2> gpurun_out/bo${v}_n4.err
done
grep -h Error gpurun_out/bo*.err | head
