# fourth session: 16-line tiles for the fused contiguous-axis spline sweeps (12 instead of 6 warps per SM):
# spline tests, config 4 A/B against VPB_SPLINE_TL=32 (the 32-line tile, same library), ncu of the x1 double sweep + density
set -x
o=gpurun_out/r02d_halftile; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_guards.py tests/test_gpu_reference_suite.py -k "spline" -x -q -p no:cacheprovider > $o/pytest_spline.log 2>&1; echo rc=$? >> $o/pytest_spline.log
timeout 900 python -m pytest tests/test_gpu_parity_headline.py tests/test_gpu_fullsize.py -k "spline or cfg4" -x -q -p no:cacheprovider -s > $o/pytest_headline.log 2>&1; echo rc=$? >> $o/pytest_headline.log
VPB_SPLINE_TL=32 timeout 900 python -m pytest tests/test_gpu_step.py -k "spline" -x -q -p no:cacheprovider > $o/pytest_spline_tl32.log 2>&1; echo rc=$? >> $o/pytest_spline_tl32.log
for i in 1 2; do
python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_tl16_$i.json 2> $o/bench_cfg4_tl16.err
VPB_SPLINE_TL=32 python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_tl32_$i.json 2> $o/bench_cfg4_tl32.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"spline_tile_kernel<1, 1, 1, 16>|spline_tile_kernel<true, true, true, 16>" --launch-skip 2 --launch-count 1 -o $o/sp_x1dbl_rho_tl16 python scripts/prof_step.py --method spline --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > $o/ncu_full_sp.log 2>&1
python scripts/ncu_kstats.py $o/sp_x1dbl_rho_tl16.ncu-rep > $o/sp_x1dbl_rho_tl16_kstats.txt 2>&1
ls -la $o
