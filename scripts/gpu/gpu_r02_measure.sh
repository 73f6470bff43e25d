# round 2: the committed measurement set (bench lines, reference arm, launch list,
# DRAM traffic per launch, emulated multi-GPU layouts).  Outputs -> gpurun_out/r02/
set -x
o=gpurun_out/r02; mkdir -p $o
python bench.py --steps 20 --warmup 5 > $o/bench_cfg2_20.json 2> $o/bench_cfg2_20.err
python bench.py > $o/bench_cfg2_default.json 2> $o/bench_cfg2_default.err
python bench.py --impl reference --steps 20 --warmup 5 > $o/ref_cfg2.json 2> $o/ref_cfg2.err
python bench.py --config cfg3 --no-cpu-baseline --e2e-steps 10 > $o/bench_cfg3.json 2> $o/bench_cfg3.err
python bench.py --config cfg4 --no-cpu-baseline --e2e-steps 10 > $o/bench_cfg4.json 2> $o/bench_cfg4.err
python bench.py --config cfg5 --no-cpu-baseline --no-e2e > $o/bench_cfg5.json 2> $o/bench_cfg5.err
python bench.py --config cfg1 --no-cpu-baseline > $o/bench_cfg1.json 2> $o/bench_cfg1.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_launch.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"dg_xcomp|dg_vplane" --launch-skip 4 --launch-count 2 --csv --log-file $o/traffic_cfg2.csv python scripts/prof_step.py --dofs 192 192 192 192 --steps 4 --advance > $o/ncu_t2.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"dg_xcomp|dg_vplane" --launch-skip 4 --launch-count 2 --csv --log-file $o/traffic_cfg5.csv python scripts/prof_step.py --dofs 288 288 288 288 --steps 4 --advance > $o/ncu_t5.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"spline_tile|density" --launch-skip 4 --launch-count 6 --csv --log-file $o/traffic_cfg4.csv python scripts/prof_step.py --method spline --order 0 --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > $o/ncu_t4.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"dg_xcomp|dg_vplane" --launch-skip 4 --launch-count 2 --csv --log-file $o/traffic_cfg3.csv python scripts/prof_step.py --problem twostream4d_baseline --order 2 --dofs 128 128 128 128 --tau 0.1 --steps 4 --advance > $o/ncu_t3.log 2>&1
python scripts/emulate_shards.py --config cfg2 --worlds 1 2 4 8 --steps 5 > $o/emu_cfg2_x1.jsonl 2>&1
python scripts/emulate_shards.py --config cfg2 --worlds 2 4 8 --steps 5 --vshard > $o/emu_cfg2_v2.jsonl 2>&1
python scripts/emulate_shards.py --config cfg5 --worlds 1 2 4 8 --steps 3 > $o/emu_cfg5_x1.jsonl 2>&1
python scripts/emulate_shards.py --config cfg5 --worlds 2 4 8 --steps 3 --vshard > $o/emu_cfg5_v2.jsonl 2>&1
ls -la $o
