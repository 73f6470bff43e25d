mkdir -p gpurun_out
P="python scripts/prof_adv.py --dofs 192 192 48 48 --steps 3"
$P > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"xplane2" -s 0 -c 1 -o gpurun_out/prof_x2s $P > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
ls -la gpurun_out
