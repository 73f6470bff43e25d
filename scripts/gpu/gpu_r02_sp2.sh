# round 2: persistent double-buffered contiguous double spline sweep
set -x
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_guards.py tests/test_gpu_parity_headline.py -q -x -m gpu -k "spline or cfg4" > gpurun_out/sp2_pytest.log 2>&1
tail -3 gpurun_out/sp2_pytest.log
for v in "" "VPB_SPLINE_DBL_BUFS=3" "VPB_SPLINE_DBL_ONESHOT=1"; do
  env $v timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sp2_bench.json 2> gpurun_out/sp2_bench.err
  echo "== $v"; python scripts/show_bench.py gpurun_out/sp2_bench.json | grep -E "value|x1x2|x2x2"
done
python scripts/xcomp_gap.py cfg2 > gpurun_out/xcomp_gap2_cfg2.json 2>&1
