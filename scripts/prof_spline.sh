mkdir -p gpurun_out
P="python scripts/prof_step.py --method spline --order 0 --dofs 128 128 64 64 --steps 1 --tau 0.1"
$P > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"spline_tile" -s 2 -c 2 -o gpurun_out/prof_sp $P > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
