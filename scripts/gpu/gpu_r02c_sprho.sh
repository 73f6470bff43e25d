# spline density epilogue in the x1 double sweep: tests and config-4 bench A/B
set -x
o=gpurun_out/r02c_sprho; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_step.py -k "spline" -x -q -p no:cacheprovider > $o/pytest_spline.log 2>&1; echo rc=$? >> $o/pytest_spline.log
timeout 900 python -m pytest tests/test_gpu_parity_headline.py -k "spline or cfg4" -x -q -p no:cacheprovider -s > $o/pytest_headline.log 2>&1; echo rc=$? >> $o/pytest_headline.log
python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_rho.json 2> $o/bench_cfg4_rho.err
VPB_SPLINE_RHO=0 python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_norho.json 2> $o/bench_cfg4_norho.err
python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_rho2.json 2> $o/bench_cfg4_rho2.err
ls -la $o
