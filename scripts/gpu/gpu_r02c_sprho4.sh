# spline: 16-byte column sums in the density epilogue, 40-point warm-up of the double recursion
set -x
o=gpurun_out/r02c_sprho4; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_guards.py -k "spline" -x -q -p no:cacheprovider > $o/pytest_spline.log 2>&1; echo rc=$? >> $o/pytest_spline.log
timeout 900 python -m pytest tests/test_gpu_parity_headline.py -k "spline or cfg4" -x -q -p no:cacheprovider -s > $o/pytest_headline.log 2>&1; echo rc=$? >> $o/pytest_headline.log
for i in 1 2; do
python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_rho$i.json 2> $o/bench_cfg4_rho.err
VPB_SPRHO_NOSUM=1 python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_nosum$i.json 2> $o/bench_cfg4_nosum.err
done
ls -la $o
