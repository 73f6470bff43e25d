# fourth session: iir_eval_fused loads the next block of points before working on the current one: tests, config 4 A/B
set -x
o=gpurun_out/r02d_prefetch; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_guards.py -k "spline" -x -q -p no:cacheprovider > $o/pytest_spline.log 2>&1; echo rc=$? >> $o/pytest_spline.log
timeout 900 python -m pytest tests/test_gpu_parity_headline.py -k "spline or cfg4" -x -q -p no:cacheprovider > $o/pytest_headline.log 2>&1; echo rc=$? >> $o/pytest_headline.log
for i in 1 2 3; do
python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_new$i.json 2> $o/bench_cfg4_new.err
VPB_LIB=vlib/libvpb200_prev.so python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_prev$i.json 2> $o/bench_cfg4_prev.err
done
ls -la $o
