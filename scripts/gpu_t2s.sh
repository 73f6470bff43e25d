mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
VPB_SPLINE_DBL_LPW2=1 timeout 600 python -m pytest tests -m gpu -x -q -k "spline_double" > gpurun_out/pytest_spl2.log 2>&1; echo pytest_lpw2_rc=$?; tail -1 gpurun_out/pytest_spl2.log
for cfg in cfg2 cfg3 cfg5; do
  for stg in 3 4 6; do
    VPB_XCOMP_STAGES=$stg timeout 300 python scripts/tune_xcomp.py --config $cfg 2>&1 | tail -1
  done
done
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_a.log 2>&1; python scripts/show_bench.py gpurun_out/bench_cfg4_a.log | head -1
VPB_SPLINE_DBL_LPW2=1 timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_b.log 2>&1; python scripts/show_bench.py gpurun_out/bench_cfg4_b.log | grep -i "value\|x1x2"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2.log 2>&1; python scripts/show_bench.py gpurun_out/bench_cfg2.log
