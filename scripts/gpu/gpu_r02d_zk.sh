# fourth session: field-solve zgemm with K staged 64 deep (2 instead of 8 stage round trips at K = 128; same k order): tests and A/B
set -x
o=gpurun_out/r02d_zk; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -k "poisson or field or solve or energy or config1 or diag" -x -q -p no:cacheprovider > $o/pytest_field.log 2>&1; echo rc=$? >> $o/pytest_field.log
for i in 1 2; do
for c in cfg3 cfg4 cfg2; do
python bench.py --config $c --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_${c}_k64_$i.json 2>> $o/err.log
VPB_LIB=vlib/libvpb200_ctma.so python bench.py --config $c --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_${c}_k16_$i.json 2>> $o/err.log
done
done
ls -la $o
