mkdir -p gpurun_out
P="python scripts/prof_step.py --dofs 192 192 48 48 --steps 2"
$P > gpurun_out/prof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_fused.csv $P > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
$P > gpurun_out/prof_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"xplane|vplane_tma|density_partial" -s 3 -c 3 -o gpurun_out/prof_fused $P > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
Q="python scripts/prof_step.py --method spline --order 0 --dofs 128 128 64 64 --steps 1 --tau 0.1"
$Q > gpurun_out/prof_plain3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"spline_tile" -s 0 -c 4 -o gpurun_out/prof_spline $Q > gpurun_out/ncu_full2.log 2>&1; echo ncu3_rc=$?
