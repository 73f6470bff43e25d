# A/B: current library vs paper_1803_02143_b200/libvpb200_old.so (alternating, same box)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "advance or composed or fullsize" > gpurun_out/pytest_ab.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_ab.log
for i in 1 2; do
for v in new old; do
  if [ $v = new ]; then L=""; else L="VPB_LIB=paper_1803_02143_b200/libvpb200_old.so"; fi
  for c in cfg2 cfg3 cfg5; do
    S=""; [ $c != cfg2 ] && S="--steps 20"
    env $L timeout 600 python bench.py --config $c $S --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$c.log 2>&1
    echo "$i $v $c $(python scripts/show_bench.py gpurun_out/ab_${v}_$c.log 2>/dev/null | grep -o 'ms/step=[0-9.]*\|sm_mhz.: [0-9.]*' | tr '\n' ' ') $(python scripts/show_bench.py gpurun_out/ab_${v}_$c.log 2>/dev/null | grep x12x12 | cut -c1-60)"
  done
done
done
