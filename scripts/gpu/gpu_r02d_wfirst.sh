# fourth session: spline tile kernels compute the evaluation weights before waiting for the tile: tests, config 4 A/B against the previous build
set -x
o=gpurun_out/r02d_wfirst2; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_guards.py tests/test_gpu_reference_suite.py -k "spline" -x -q -p no:cacheprovider > $o/pytest_spline.log 2>&1; echo rc=$? >> $o/pytest_spline.log
timeout 900 python -m pytest tests/test_gpu_parity_headline.py tests/test_gpu_fullsize.py -k "spline or cfg4" -x -q -p no:cacheprovider > $o/pytest_headline.log 2>&1; echo rc=$? >> $o/pytest_headline.log
for i in 1 2 3; do
python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_new$i.json 2> $o/bench_cfg4_new.err
VPB_LIB=vlib/libvpb200_wfirst.so python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_base$i.json 2> $o/bench_cfg4_base.err
done
ls -la $o
