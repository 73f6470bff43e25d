mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log; grep -B5 "Error" gpurun_out/pytest_gpu.log | head -30
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.log 2>&1; echo cfg4_rc=$?; python scripts/show_bench.py gpurun_out/bench_cfg4.log
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2.log 2>&1; echo cfg2_rc=$?; python scripts/show_bench.py gpurun_out/bench_cfg2.log
