# double-x-pass validation + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "advance or double_x or sparse_diag" > gpurun_out/pytest_adv.log 2>&1; echo pytest_adv_rc=$?; tail -15 gpurun_out/pytest_adv.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_adv.log 2>&1; echo bench_rc=$?; python scripts/show_bench.py gpurun_out/bench_adv.log; python -c "import json;d=json.loads(open('gpurun_out/bench_adv.log').read().strip().splitlines()[-1]);print('per_call',d['per_call'])"
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_adv3.log 2>&1; echo bench3_rc=$?; python scripts/show_bench.py gpurun_out/bench_adv3.log
