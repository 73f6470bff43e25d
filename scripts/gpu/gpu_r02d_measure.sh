# fourth-session (final) measurement set at HEAD: bench lines of configs 1-5 (driver
# command and BASELINE step counts; config 5 now with e2e), the reference arm, the ncu
# launch list of the driver command, per-launch DRAM traffic at configs 2 and 4, one
# --set full capture each of the composed x pass and of the spline x1 double sweep + density
set -x
o=gpurun_out/r02d_meas; mkdir -p $o
python bench.py --steps 20 --warmup 5 > $o/bench_cfg2_20.json 2> $o/bench_cfg2_20.err
python bench.py > $o/bench_cfg2_default.json 2> $o/bench_cfg2_default.err
python bench.py --config cfg3 --no-cpu-baseline --e2e-steps 10 > $o/bench_cfg3.json 2> $o/bench_cfg3.err
python bench.py --config cfg4 --no-cpu-baseline --e2e-steps 10 > $o/bench_cfg4.json 2> $o/bench_cfg4.err
python bench.py --config cfg5 --no-cpu-baseline --e2e-steps 3 > $o/bench_cfg5.json 2> $o/bench_cfg5.err
python bench.py --config cfg1 --no-cpu-baseline > $o/bench_cfg1.json 2> $o/bench_cfg1.err
python bench.py --impl reference --steps 20 --warmup 5 > $o/bench_reference_cfg2.json 2> $o/bench_reference_cfg2.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o/plain_launch.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_launch.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"dg_xcomp|dg_vplane" --launch-skip 4 --launch-count 2 --csv --log-file $o/traffic_cfg2.csv python scripts/prof_step.py --dofs 192 192 192 192 --steps 4 --advance > $o/ncu_t2.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"spline_tile" --launch-skip 8 --launch-count 4 --csv --log-file $o/traffic_cfg4.csv python scripts/prof_step.py --method spline --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > $o/ncu_t4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dg_xcomp --launch-skip 2 --launch-count 1 -o $o/xcomp_cfg2 python scripts/prof_adv.py --dofs 192 192 192 192 --steps 4 > $o/ncu_full_xcomp.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"spline_tile_kernel<true, true, true>|spline_tile_kernel<1, 1, 1>" --launch-skip 2 --launch-count 1 -o $o/sp_x1dbl_rho python scripts/prof_step.py --method spline --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > $o/ncu_full_sp.log 2>&1
for r in xcomp_cfg2 sp_x1dbl_rho; do python scripts/ncu_kstats.py $o/$r.ncu-rep > $o/${r}_kstats.txt 2>&1; done
ls -la $o
