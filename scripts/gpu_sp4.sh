mkdir -p gpurun_out
for v in cur rows3 rows4; do if [ $v != cur ]; then export VPB_LIB=$PWD/ab/libvpb200_$v.so; fi
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bsp_$v.log 2>&1; echo "== $v"; python scripts/show_bench.py gpurun_out/bsp_$v.log | grep -E "x1|value" | cut -c1-120; done
