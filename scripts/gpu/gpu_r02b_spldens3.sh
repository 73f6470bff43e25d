# ncu of the spline x2 double sweep with / without the cluster density epilogue (config 4)
set -x
o=gpurun_out/r02b_spd3; mkdir -p $o
P="python scripts/prof_step.py --method spline --order 0 --dofs 128 128 128 128 --tau 0.1 --steps 3 --advance"
$P > $o/plain.log 2>&1 && VPB_FUSE_RHO=0 $P > $o/plain0.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spline_tile_kernel" --launch-skip 5 --launch-count 1 -o $o/prof_rho $P > $o/ncu.log 2>&1; \
VPB_FUSE_RHO=0 ncu --set full --clock-control none --import-source on -k regex:"spline_tile_kernel" --launch-skip 5 --launch-count 1 -o $o/prof_sep $P > $o/ncu0.log 2>&1; echo ncu_rc=$?
ls $o
