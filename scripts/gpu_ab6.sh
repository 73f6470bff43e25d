mkdir -p gpurun_out
run() { name=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${name}_$C.log 2>&1; echo "== $name $C"; python scripts/show_bench.py gpurun_out/ab_${name}_$C.log | grep -E "x12x12|value" | cut -c1-110; }
C=cfg2
for r in 1 2; do
run cur VPB_X=1
run direct VPB_LIB=$PWD/ab/libvpb200_direct.so VPB_XPLANE2_STAGES=4
done
