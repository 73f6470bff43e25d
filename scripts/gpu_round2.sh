# tests, smoke, default bench (e2e + cpu baseline), cfg3/cfg5/cfg4 lines, ncu launch list of the bench command
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?; python scripts/show_bench.py gpurun_out/bench.log
for c in cfg3 cfg5 cfg4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; echo bench_${c}_rc=$?; python scripts/show_bench.py gpurun_out/bench_$c.log; done
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/bench_plain_for_ncu.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_cfg2.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
