# fourth session, final check at HEAD: smoke, the whole -m gpu suite, the driver's bench command, the opt-in config-5 parity test
set -x
o=gpurun_out/r02d_final; mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo smoke rc=$? >> $o/smoke.log
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/pytest_gpu.log 2>&1; echo rc=$? >> $o/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > $o/bench_cfg2_20.json 2> $o/bench_cfg2_20.err
ls -la $o
