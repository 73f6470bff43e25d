# xcomp running-sum rewrite: bitwise digest and timing vs the previous build
# (vlib/libvpb200_old.so), then the sharded solvers through NCCL at one rank
set -x
o=gpurun_out/r02b_ab; mkdir -p $o
python scripts/xcomp_digest.py > $o/digest_new.json 2>&1
VPB_LIB=vlib/libvpb200_old.so python scripts/xcomp_digest.py > $o/digest_old.json 2>&1
for c in cfg2 cfg5 cfg3; do
  for rep in 1 2; do
    VPB_LIB=vlib/libvpb200_old.so python scripts/tune_xcomp.py --config $c --reps 9 >> $o/tune_old.jsonl 2>&1
    python scripts/tune_xcomp.py --config $c --reps 9 >> $o/tune_new.jsonl 2>&1
  done
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "xcomp or advance or fast or headline or shard or dist" > $o/pytest_sub.log 2>&1; echo rc=$? >> $o/pytest_sub.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $o/bench_new.json 2> $o/bench_new.err
VPB_LIB=vlib/libvpb200_old.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $o/bench_old.json 2> $o/bench_old.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $o/bench_new2.json 2> $o/bench_new2.err
timeout 600 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --steps 10 --warmup 3 > $o/sharded_v.json 2> $o/sharded_v.err
timeout 600 python bench.py --sharded --steps 10 --warmup 3 --layout v --peer-halos > $o/sharded_vpeer.json 2> $o/sharded_vpeer.err
timeout 600 python bench.py --sharded --steps 10 --warmup 3 --layout x > $o/sharded_x.json 2> $o/sharded_x.err
timeout 600 python bench.py --sharded --steps 10 --warmup 3 --config cfg4 > $o/sharded_spline.json 2> $o/sharded_spline.err
timeout 600 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29532 bench.py --sharded --steps 10 --warmup 3 > $o/sharded_v_torchrun.json 2> $o/sharded_v_torchrun.err
ls -la $o
