mkdir -p gpurun_out
P="python scripts/prof_step.py --dofs 192 192 48 48 --steps 2"
$P > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"xplane|vplane_tma" -s 3 -c 3 -o gpurun_out/prof_rho $P > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
