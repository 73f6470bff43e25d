mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -x -q -k "spline" > gpurun_out/pytest_sp.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_sp.log
VPB_SPLINE_LPW=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "spline_pcr" > gpurun_out/pytest_sp1.log 2>&1; echo pytest_lpw1_rc=$?; tail -1 gpurun_out/pytest_sp1.log
for v in 2 1; do
VPB_SPLINE_LPW=$v timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bsp_$v.log 2>&1; echo "== lpw $v"; python scripts/show_bench.py gpurun_out/bsp_$v.log | grep -E "x1|value" | cut -c1-120; done
