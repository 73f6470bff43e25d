mkdir -p gpurun_out
VPB_LIB=$PWD/ab/libvpb200_fma.so timeout 600 python -m pytest tests/test_gpu_step.py -q -k "golden or config1" > gpurun_out/pytest_fma.log 2>&1; echo pytest_fma_rc=$?; tail -1 gpurun_out/pytest_fma.log
run() { name=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${name}_$C.log 2>&1; echo "== $name $C"; python scripts/show_bench.py gpurun_out/ab_${name}_$C.log | grep -E "sweep|value" | cut -c1-110; }
for C in cfg2 cfg3; do for r in 1 2; do
run exact VPB_X=1
run fma VPB_LIB=$PWD/ab/libvpb200_fma.so
done; done
