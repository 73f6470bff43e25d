mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "spline or plugin or steps_match or cfg4 or reduced" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.log 2>&1; echo bench_rc=$?
