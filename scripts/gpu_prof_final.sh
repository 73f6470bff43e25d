# launch list of advance() at full config 2 + --set full of the double x pass (reduced v grid)
mkdir -p gpurun_out
P="python scripts/prof_adv.py --dofs 192 192 192 192 --steps 3"
$P > gpurun_out/prof_full_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_adv_cfg2.csv $P > gpurun_out/ncu_l.log 2>&1; echo ncu1_rc=$?
Q="python scripts/prof_adv.py --dofs 192 192 48 48 --steps 3"
$Q > gpurun_out/prof_red_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"xplane2" -s 0 -c 1 -o gpurun_out/prof_x2_final $Q > gpurun_out/ncu_f.log 2>&1; echo ncu2_rc=$?
