# composed-pass register cap A/B (sustained 100-step config 2 runs, alternating)
mkdir -p gpurun_out
for i in 1 2; do
for v in base r192 r176; do
  if [ $v = base ]; then L=""; else L="VPB_LIB=paper_1803_02143_b200/libvpb200_$v.so"; fi
  env $L timeout 600 python bench.py --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_rc_$v.log 2>&1
  echo "$v: $(python scripts/show_bench.py gpurun_out/bench_rc_$v.log 2>/dev/null | grep -o 'ms/step=[0-9.]*\|sm_mhz.: [0-9.]*' | tr '\n' ' ') $(python scripts/show_bench.py gpurun_out/bench_rc_$v.log 2>/dev/null | grep x12x12)"
done
done
for v in r192 r176; do VPB_LIB=paper_1803_02143_b200/libvpb200_$v.so timeout 300 python scripts/tune_xcomp.py --config cfg5 2>&1 | tail -1; done
timeout 300 python scripts/tune_xcomp.py --config cfg5 2>&1 | tail -1
