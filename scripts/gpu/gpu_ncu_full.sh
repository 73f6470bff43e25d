# one --set full capture of the step's two hot passes at the full config-2 size
mkdir -p gpurun_out
P="python scripts/prof_adv.py --dofs 192 192 192 192 --steps 2"
$P > gpurun_out/prof_plain_full.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"xcomp|vplane_tma" -c 3 -o gpurun_out/prof_cfg2_full $P > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_full.log
