# x-plane dof-split: correctness + A/B of register budgets vs the previous design
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
for c in cfg2 cfg3; do
for v in cur r96 r128 head; do
  if [ $v = cur ]; then L=""; else L=$PWD/ab/libvpb200_$v.so; fi
  VPB_LIB=$L timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$c.log 2>&1
  echo "== $v $c"; python scripts/show_bench.py gpurun_out/ab_${v}_$c.log | grep -E "sweep|value"
done; done
