mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -x -q -k "spline" > gpurun_out/pytest_sp.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_sp.log
for v in iir pcr; do if [ $v = pcr ]; then export VPB_SPLINE_PCR=1; fi
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bsp_$v.log 2>&1; echo "== $v"; python scripts/show_bench.py gpurun_out/bsp_$v.log | cut -c1-120; done
