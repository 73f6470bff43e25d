# round 2: fused evaluation + bulk write-out for single contiguous spline sweeps too
set -x
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_guards.py tests/test_gpu_parity_headline.py tests/test_gpu_reference_suite.py -q -x -m gpu -k "spline or cfg4 or suite or landau2d" > gpurun_out/sp5_pytest.log 2>&1
tail -2 gpurun_out/sp5_pytest.log
for v in "" "VPB_SPLINE_ROWS=1"; do
  env $v timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --per-step > gpurun_out/sp5_bench.json 2> gpurun_out/sp5_bench.err
  echo "== per-step $v"; python scripts/show_bench.py gpurun_out/sp5_bench.json | grep -E "value|sweep_x"
done
