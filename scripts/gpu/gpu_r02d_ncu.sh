# fourth session: one --set full capture per dominant kernel at HEAD (v-plane pass at config 2; the four spline tile sweeps of a config-4 step)
set -x
o=gpurun_out/r02d_ncu; mkdir -p $o
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dg_vplane --launch-skip 2 --launch-count 1 -o $o/vplane_cfg2 python scripts/prof_adv.py --dofs 192 192 192 192 --steps 4 > $o/ncu_vplane.log 2>&1
# spline advance(5): launches of spline_tile_kernel: x1, x2 (open), then per step v1, v2, x2x2, x1x1+rho
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spline_tile --launch-skip 8 --launch-count 4 -o $o/spline_cfg4 python scripts/prof_step.py --method spline --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > $o/ncu_spline.log 2>&1
for r in vplane_cfg2 spline_cfg4; do python scripts/ncu_kstats.py $o/$r.ncu-rep > $o/${r}_kstats.txt 2>&1; done
ls -la $o
