mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py -x -q -k "fused_v or vplane or nonfinite or config1 or advance_bitwise" > gpurun_out/pytest_v.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_v.log
P="python scripts/prof_adv.py --dofs 192 192 192 192 --steps 2"
$P > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"vplane" --csv --log-file gpurun_out/l_v.csv $P > /dev/null 2>&1; echo ncu_rc=$?
run() { name=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${name}_$C.log 2>&1; echo "== $name $C"; python scripts/show_bench.py gpurun_out/ab_${name}_$C.log | grep -E "v12|value" | cut -c1-110; }
for C in cfg2 cfg3 cfg5; do for r in 1 2; do
run win VPB_X=1
run base VPB_LIB=$PWD/ab/libvpb200_base.so
done; done
