mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "spline" > gpurun_out/pytest_spl.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_spl.log
VPB_SPLINE_DBL_LPW2=1 timeout 600 python -m pytest tests -m gpu -x -q -k "spline_double" > gpurun_out/pytest_spl2.log 2>&1; echo pytest2_rc=$?; tail -2 gpurun_out/pytest_spl2.log
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_a.log 2>&1; python scripts/show_bench.py gpurun_out/bench_cfg4_a.log | head -8
VPB_SPLINE_DBL_LPW2=1 timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_b.log 2>&1; python scripts/show_bench.py gpurun_out/bench_cfg4_b.log | head -8
