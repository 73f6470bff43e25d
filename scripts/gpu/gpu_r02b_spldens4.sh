# spline x2 density epilogue with the tile written after the cluster barrier:
# tests + config 4 bench A/B + ncu of the fused launch
set -x
o=gpurun_out/r02b_spd4; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_guards.py -m gpu -x -q -p no:cacheprovider -k "spline or bounds" > $o/pytest_spline.log 2>&1; echo rc=$? >> $o/pytest_spline.log
for rep in 1 2; do
  python bench.py --config cfg4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $o/fused$rep.json 2> $o/fused$rep.err
  VPB_FUSE_RHO=0 python bench.py --config cfg4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $o/sep$rep.json 2> $o/sep$rep.err
done
P="python scripts/prof_step.py --method spline --order 0 --dofs 128 128 128 128 --tau 0.1 --steps 3 --advance"
$P > $o/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spline_tile_kernel" --launch-skip 5 --launch-count 1 -o $o/prof_rho $P > $o/ncu.log 2>&1; echo ncu_rc=$?
ls $o
