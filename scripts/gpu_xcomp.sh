# composed merged x pass: GPU tests, fast vs exact bench lines at cfg2/3/5
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
for c in cfg2 cfg3 cfg5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_fast_$c.log 2>&1; echo fast_${c}_rc=$?; python scripts/show_bench.py gpurun_out/bench_fast_$c.log
done
VPB_ARITH=exact timeout 900 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_exact_cfg2.log 2>&1; echo exact_rc=$?; python scripts/show_bench.py gpurun_out/bench_exact_cfg2.log
