mkdir -p gpurun_out
VPB_LIB=$PWD/ab/libvpb200_direct.so timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "advance or double_x" > gpurun_out/pytest_direct.log 2>&1; echo pytest_direct_rc=$?; tail -1 gpurun_out/pytest_direct.log
run() { name=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${name}_$C.log 2>&1; echo "== $name $C"; python scripts/show_bench.py gpurun_out/ab_${name}_$C.log | grep -E "x12x12|value" | cut -c1-110; }
for C in cfg2 cfg3; do
run base VPB_LIB=$PWD/ab/libvpb200_base.so
run direct VPB_LIB=$PWD/ab/libvpb200_direct.so
run direct_g1 VPB_LIB=$PWD/ab/libvpb200_direct.so VPB_XPLANE2_CHUNK=4608
run direct_s2 VPB_LIB=$PWD/ab/libvpb200_direct.so VPB_XPLANE2_STAGES=2
run direct_s4 VPB_LIB=$PWD/ab/libvpb200_direct.so VPB_XPLANE2_STAGES=4
run base_s2 VPB_LIB=$PWD/ab/libvpb200_base.so VPB_XPLANE2_STAGES=2
done
