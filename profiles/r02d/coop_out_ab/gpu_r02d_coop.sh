# fourth session: fused contiguous spline sweeps write out by the whole warp (16 B per lane) with the density riding on the same loads: tests, config 4 A/B
set -x
o=gpurun_out/r02d_coop; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_guards.py tests/test_gpu_reference_suite.py -k "spline" -x -q -p no:cacheprovider > $o/pytest_spline.log 2>&1; echo rc=$? >> $o/pytest_spline.log
timeout 900 python -m pytest tests/test_gpu_parity_headline.py tests/test_gpu_fullsize.py -k "spline or cfg4" -x -q -p no:cacheprovider > $o/pytest_headline.log 2>&1; echo rc=$? >> $o/pytest_headline.log
for i in 1 2 3; do
python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_coop$i.json 2> $o/bench_cfg4_coop.err
VPB_SPLINE_COOP_OUT=0 python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_bulk$i.json 2> $o/bench_cfg4_bulk.err
done
ls -la $o
