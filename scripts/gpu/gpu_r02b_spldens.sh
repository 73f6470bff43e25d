# spline x2 double sweep with the cluster density epilogue: tests, config 4
# bench loop vs the standalone density pass (VPB_FUSE_RHO=0), guard bands
set -x
o=gpurun_out/r02b_spd; mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_guards.py -m gpu -x -q -p no:cacheprovider -k "spline or guard or bounds or density" > $o/pytest_spline.log 2>&1; echo rc=$? >> $o/pytest_spline.log
for rep in 1 2; do
  python bench.py --config cfg4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $o/fused$rep.json 2> $o/fused$rep.err
  VPB_FUSE_RHO=0 python bench.py --config cfg4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $o/sep$rep.json 2> $o/sep$rep.err
done
timeout 1500 python -m pytest tests/test_gpu_parity_headline.py -m gpu -q -p no:cacheprovider -k "spline" > $o/pytest_headline_spline.log 2>&1; echo rc=$? >> $o/pytest_headline_spline.log
ls $o
