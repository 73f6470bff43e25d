# default bench (recorded), cfg3/cfg5/cfg4/cfg1 lines
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?; python scripts/show_bench.py gpurun_out/bench.log
for c in cfg3 cfg5 cfg4 cfg1; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; echo bench_${c}_rc=$?; done
P="python scripts/prof_adv.py --dofs 192 192 48 48 --steps 3"
$P > gpurun_out/prof_plain2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_adv.csv $P > gpurun_out/ncu_launch.log 2>&1; echo ncu2_rc=$?
