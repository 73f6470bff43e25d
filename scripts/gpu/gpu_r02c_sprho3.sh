# spline density epilogue A/B: column sums on / off (tile mapping alone)
set -x
o=gpurun_out/r02c_sprho3; mkdir -p $o
for i in 1 2; do
python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_rho$i.json 2> $o/bench_cfg4_rho.err
VPB_SPRHO_NOSUM=1 python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_nosum$i.json 2> $o/bench_cfg4_nosum.err
done
ls -la $o
