# A/B: current build vs ab/libvpb200_head.so, alternating, cfg2 + cfg3
mkdir -p gpurun_out
for r in 1 2; do
for c in cfg3 cfg2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_new_${c}_$r.log 2>&1
  VPB_LIB=$PWD/ab/libvpb200_head.so timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_old_${c}_$r.log 2>&1
  for v in new old; do echo "$v $c $r"; python scripts/show_bench.py gpurun_out/ab_${v}_${c}_$r.log | grep -E "sweep|value"; done
done; done
