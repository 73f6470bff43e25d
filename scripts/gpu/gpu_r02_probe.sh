set -x
python scripts/pcie_probe.py > gpurun_out/pcie_probe.json 2>&1
python scripts/e2e_sweep.py 4 8 16 32 64 > gpurun_out/e2e_sweep.txt 2>&1
python scripts/xcomp_gap.py cfg2 > gpurun_out/xcomp_gap_cfg2.json 2>&1
python scripts/xcomp_gap.py cfg5 > gpurun_out/xcomp_gap_cfg5.json 2>&1
python -m pytest tests/test_gpu_parity_headline.py tests/test_gpu_snapshots.py tests/test_gpu_dist.py -q -s -m gpu > gpurun_out/parity2.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:spline_tile_kernel<true, true, true>' --launch-skip 2 --launch-count 1 -o gpurun_out/ncu_spline_x1dbl -f python scripts/prof_step.py --method spline --order 0 --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > gpurun_out/ncu_spline.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:dg_xcomp_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/ncu_xcomp_cfg5geom -f python scripts/prof_step.py --method dg --order 3 --dofs 288 288 48 48 --tau 0.05 --steps 5 --advance > gpurun_out/ncu_xcomp.log 2>&1
