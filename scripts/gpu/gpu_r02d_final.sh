# fourth session, final check at HEAD: smoke, the whole -m gpu suite, the driver's bench command, config 4's bench line
set -x
o=gpurun_out/r02d_final2; mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo smoke rc=$? >> $o/smoke.log
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/pytest_gpu.log 2>&1; echo rc=$? >> $o/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > $o/bench_cfg2_20.json 2> $o/bench_cfg2_20.err
python bench.py --config cfg4 --no-cpu-baseline --e2e-steps 10 > $o/bench_cfg4.json 2> $o/bench_cfg4.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"spline_tile" --launch-skip 8 --launch-count 4 --csv --log-file $o/traffic_cfg4.csv python scripts/prof_step.py --method spline --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > $o/ncu_t4.log 2>&1
ls -la $o
