# one gpurun call: tests, bench, launch list, one full ncu capture
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_rc=$?
for c in cfg3 cfg4 cfg1; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; echo bench_${c}_rc=$?; done
P="python scripts/prof_step.py --dofs 192 192 48 48 --steps 2"
$P > gpurun_out/prof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
$P > gpurun_out/prof_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"dg_rows|dg_cols|density_partial" -s 3 -c 4 -o gpurun_out/prof_r01 $P > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
