# blocked v->x step: tests, then A/B bench at cfg2/cfg3/cfg5 with VPB_VX=0/1 and block shapes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "vx or advance or composed" > gpurun_out/pytest_vx.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/pytest_vx.log
for c in cfg2; do
  for nb in "8 2" "4 2" "8 4" "4 4" "16 1"; do
    set -- $nb
    VPB_VX=1 VPB_VX_NB1=$1 VPB_VX_NB2=$2 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_vx_${c}_$1_$2.log 2>&1; echo vx_${c}_$1_$2 rc=$?; python scripts/show_bench.py gpurun_out/bench_vx_${c}_$1_$2.log
  done
done
