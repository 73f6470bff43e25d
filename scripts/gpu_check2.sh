mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; cat gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2.log 2>&1; python scripts/show_bench.py gpurun_out/bench_cfg2.log
S=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$? $(( $(date +%s)-S ))s; tail -c 1500 gpurun_out/bench_ref.log
