# round 2: fused contiguous double spline sweep (solve + evaluation, staggered lanes)
set -x
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_guards.py tests/test_gpu_parity_headline.py -q -x -m gpu -k "spline or cfg4" > gpurun_out/sp1_pytest.log 2>&1
tail -3 gpurun_out/sp1_pytest.log
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sp1_bench_cfg4.json 2> gpurun_out/sp1_bench_cfg4.err
python scripts/show_bench.py gpurun_out/sp1_bench_cfg4.json
ncu --set full --import-source on --clock-control none -k regex:spline_tile_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/ncu_spline_x1dbl_v2 -f python scripts/prof_step.py --method spline --order 0 --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > gpurun_out/ncu_spline2.log 2>&1
