# ncu --set full of the spline step kernels at the full config-4 size (advance: double x sweeps)
mkdir -p gpurun_out
P="python scripts/prof_adv.py --problem landau4d --method spline --dofs 128 128 128 128 --steps 2 --tau 0.1"
$P > gpurun_out/prof_plain_spline.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"spline_rows|spline_tile" -c 6 -o gpurun_out/prof_cfg4_full $P > gpurun_out/ncu_spline.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_spline.log
