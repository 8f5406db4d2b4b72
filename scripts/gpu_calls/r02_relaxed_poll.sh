# A/B of the barrier poll: acquire loads (default) vs relaxed loads + one acquire fence
set -x
for v in default relaxed; do
  if [ $v = relaxed ]; then export MGWFBP_B200_LIB=$PWD/paper_1811_11141_b200/_lib/libmgwfbp_b200_relaxed.so; else unset MGWFBP_B200_LIB; fi
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2956${#v} scripts/phase_probe.py > gpurun_out/phases_n4_$v.json 2> gpurun_out/phases_n4_$v.err
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2957${#v} scripts/algo_sweep.py --mib 1,2,4,8,16,32 --algos oneshot,twoshot,push,push_oneshot,auto > gpurun_out/sweep_n4_$v.json 2> gpurun_out/sweep_n4_$v.err
done
tail -n 2 gpurun_out/*.err
