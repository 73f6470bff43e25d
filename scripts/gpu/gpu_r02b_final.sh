# final verification of the second session: smoke, the whole -m gpu suite,
# the driver's bench commands (ours and the reference arm), e2e step scaling
set -x
o=gpurun_out/r02b_final; mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo smoke rc=$? >> $o/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/pytest_gpu.log 2>&1; echo rc=$? >> $o/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > $o/bench_cfg2_20.json 2> $o/bench_cfg2_20.err
python bench.py --impl reference --steps 20 --warmup 5 > $o/ref_cfg2.json 2> $o/ref_cfg2.err
python scripts/e2e_steps.py 16 > $o/e2e_steps16.json 2>&1
ls -la $o
