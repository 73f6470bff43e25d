# round 2: contiguous double spline sweep without wrap arithmetic; full GPU suite
set -x
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sp3_bench.json 2> gpurun_out/sp3_bench.err
python scripts/show_bench.py gpurun_out/sp3_bench.json
ncu --set full --import-source on --clock-control none -k regex:spline_tile_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/ncu_spline_x1dbl_v3 -f python scripts/prof_step.py --method spline --order 0 --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > gpurun_out/ncu_spline3.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/full_gpu_pytest.log 2>&1
tail -3 gpurun_out/full_gpu_pytest.log
