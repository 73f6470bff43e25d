mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
for nb in "8 4" "4 8"; do
  set -- $nb
  VPB_VX=1 VPB_VX_NB1=$1 VPB_VX_NB2=$2 timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_vx_cfg3_$1_$2.log 2>&1; echo vx_cfg3_$1_$2 rc=$?; python scripts/show_bench.py gpurun_out/bench_vx_cfg3_$1_$2.log
done
