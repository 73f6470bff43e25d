# steady-state interleaved double pass vs base
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "advance or double_x or sparse_diag" > gpurun_out/pytest_adv.log 2>&1; echo pytest_adv_rc=$?; tail -1 gpurun_out/pytest_adv.log
for r in 1 2; do
for c in cfg2 cfg3; do
for v in cur base; do
  if [ $v = cur ]; then L=""; else L=$PWD/ab/libvpb200_$v.so; fi
  VPB_LIB=$L timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$c.log 2>&1
  echo "== $v $c"; python scripts/show_bench.py gpurun_out/ab_${v}_$c.log | grep -E "sweep_x12x12|value"
done; done; done
