# round 2: xcomp T2S A/B, e2e timeline, spline x1 ncu, new GPU tests
set -x
for cfg in cfg2 cfg3 cfg5; do
  timeout 300 python scripts/tune_xcomp.py --config $cfg 2>&1 | tail -1
  VPB_LIB=ab/libvpb200_t2s.so timeout 300 python scripts/tune_xcomp.py --config $cfg 2>&1 | tail -1
done > gpurun_out/ab_t2s.txt
VPB_LIB=ab/libvpb200_t2s.so timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py -q -x -m gpu -k "advance or fast or fullsize" > gpurun_out/ab_t2s_pytest.log 2>&1
python scripts/e2e_timeline.py 16 > gpurun_out/e2e_timeline.json 2>&1
timeout 1200 python -m pytest tests/test_gpu_snapshots.py tests/test_gpu_guards.py tests/test_gpu_reference_suite.py -q -m gpu > gpurun_out/new_tests.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:spline_tile_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/ncu_spline_x1dbl -f python scripts/prof_step.py --method spline --order 0 --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > gpurun_out/ncu_spline.log 2>&1
