mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k "advance or double_x or sparse_diag" > gpurun_out/pytest_adv.log 2>&1; echo pytest_adv_rc=$?; tail -2 gpurun_out/pytest_adv.log
P="python scripts/prof_adv.py --dofs 192 192 48 48 --steps 3"
$P > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"xplane2" -s 0 -c 1 -o gpurun_out/prof_x2 $P > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
