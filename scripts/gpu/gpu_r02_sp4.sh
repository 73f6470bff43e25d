# round 2: bulk-store writeout of the contiguous double spline sweep; xcomp T2S only for 3-warp CTAs
set -x
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_guards.py tests/test_gpu_parity_headline.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x -m gpu > gpurun_out/sp4_pytest.log 2>&1
tail -2 gpurun_out/sp4_pytest.log
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sp4_bench.json 2> gpurun_out/sp4_bench.err
python scripts/show_bench.py gpurun_out/sp4_bench.json
for cfg in cfg2 cfg5; do timeout 300 python scripts/tune_xcomp.py --config $cfg 2>&1 | tail -1; done
ncu --set full --import-source on --clock-control none -k regex:spline_tile_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/ncu_spline_x1dbl_v4 -f python scripts/prof_step.py --method spline --order 0 --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > gpurun_out/ncu_spline4.log 2>&1
