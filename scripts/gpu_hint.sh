mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k "advance or density or fused_x" > gpurun_out/pytest_h.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_h.log
P="python scripts/prof_adv.py --dofs 192 192 192 192 --steps 3"
$P > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"xplane" --csv --log-file gpurun_out/l_hint.csv $P > /dev/null 2>&1; echo ncu_rc=$?
run() { name=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${name}_$C.log 2>&1; echo "== $name $C"; python scripts/show_bench.py gpurun_out/ab_${name}_$C.log | grep -E "x12|value" | cut -c1-110; }
for C in cfg2 cfg3; do for r in 1 2; do
run hint VPB_X=1
run nohint VPB_LIB=$PWD/ab/libvpb200_nohint.so
done; done
