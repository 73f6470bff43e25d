# fourth session: smoke, the whole -m gpu suite and the bench of every config at HEAD (fresh build)
set -x
o=gpurun_out/r02d_check; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $o/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo smoke rc=$? >> $o/smoke.log
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/pytest_gpu.log 2>&1; echo rc=$? >> $o/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > $o/bench_cfg2_20.json 2> $o/bench_cfg2_20.err
for c in cfg3 cfg4 cfg5 cfg1; do
python bench.py --config $c --warmup 5 --no-cpu-baseline > $o/bench_$c.json 2> $o/bench_$c.err
done
ls -la $o
