# one gpurun call: GPU tests + cfg2/cfg3 bench (no cpu baseline / e2e)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
for c in cfg2 cfg3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; echo bench_${c}_rc=$?; python scripts/show_bench.py gpurun_out/bench_$c.log; done
