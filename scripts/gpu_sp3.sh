mkdir -p gpurun_out
for v in rows tiles; do if [ $v = tiles ]; then export VPB_SPLINE_TILES=1; fi
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bsp_$v.log 2>&1; echo "== $v"; python scripts/show_bench.py gpurun_out/bsp_$v.log | cut -c1-120; done
