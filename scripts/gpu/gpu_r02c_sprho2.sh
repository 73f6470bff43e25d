# spline density epilogue, column sums with register accumulators: tests and config-4 bench
set -x
o=gpurun_out/r02c_sprho2; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_step.py -k "spline" -x -q -p no:cacheprovider > $o/pytest_spline.log 2>&1; echo rc=$? >> $o/pytest_spline.log
python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_rho.json 2> $o/bench_cfg4_rho.err
VPB_SPLINE_RHO=0 python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_norho.json 2> $o/bench_cfg4_norho.err
ls -la $o
