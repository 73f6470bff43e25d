# A/B: density epilogue on/off, cfg2 + cfg3, alternating; then the density tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k "density or fused or neutral or nonfinite" > gpurun_out/pytest_rho.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_rho.log
for r in 1 2; do
for c in cfg2 cfg3; do
  for v in 0 1; do
  VPB_FUSE_RHO=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rho${v}_${c}_$r.log 2>&1
  echo "rho=$v $c $r"; python scripts/show_bench.py gpurun_out/rho${v}_${c}_$r.log | grep -E "sweep|value|density"
  done
done; done
