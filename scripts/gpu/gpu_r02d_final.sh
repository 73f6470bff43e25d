# fourth session, final check at HEAD: smoke, the whole -m gpu suite, the driver's bench command, configs 3 and 4
set -x
o=gpurun_out/r02d_final4; mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo smoke rc=$? >> $o/smoke.log
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/pytest_gpu.log 2>&1; echo rc=$? >> $o/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > $o/bench_cfg2_20.json 2> $o/bench_cfg2_20.err
python bench.py --config cfg4 --no-cpu-baseline --e2e-steps 10 > $o/bench_cfg4.json 2> $o/bench_cfg4.err
python bench.py --config cfg3 --no-cpu-baseline --e2e-steps 10 > $o/bench_cfg3.json 2> $o/bench_cfg3.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"spline_tile" --launch-skip 8 --launch-count 4 --csv --log-file $o/traffic_cfg4.csv python scripts/prof_step.py --method spline --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > $o/ncu_t4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spline_tile --launch-skip 9 --launch-count 1 -o $o/sp_x1dbl_rho python scripts/prof_step.py --method spline --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > $o/ncu_full_sp.log 2>&1
python scripts/ncu_kstats.py $o/sp_x1dbl_rho.ncu-rep > $o/sp_x1dbl_rho_kstats.txt 2>&1
ls -la $o
