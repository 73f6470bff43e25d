# third session: smoke, the whole -m gpu suite and the driver's bench command at HEAD
set -x
o=gpurun_out/r02c_check; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $o/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo smoke rc=$? >> $o/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/pytest_gpu.log 2>&1; echo rc=$? >> $o/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > $o/bench_cfg2_20.json 2> $o/bench_cfg2_20.err
ls -la $o
