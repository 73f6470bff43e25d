# one gpurun call: GPU tests, default bench, graph-replay benches
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --graph --no-cpu-baseline --no-e2e > gpurun_out/bench_graph.log 2>&1; echo bench_graph_rc=$?
for c in cfg1 cfg4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; echo bench_${c}_rc=$?;
 timeout 600 python bench.py --config $c --steps 20 --warmup 3 --graph --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_graph.log 2>&1; echo bench_${c}_graph_rc=$?; done
