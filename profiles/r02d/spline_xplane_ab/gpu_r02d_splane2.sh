# fourth session: segmented one-kernel merged spline x pass: tests, config 4 A/B (segmented / whole lines / two passes), ncu
set -x
o=gpurun_out/r02d_splane3; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_guards.py -k "spline" -q -p no:cacheprovider > $o/pytest_spline.log 2>&1; echo rc=$? >> $o/pytest_spline.log
timeout 900 python -m pytest tests/test_gpu_parity_headline.py tests/test_gpu_fullsize.py -k "spline or cfg4" -x -q -p no:cacheprovider -s > $o/pytest_headline.log 2>&1; echo rc=$? >> $o/pytest_headline.log
for i in 1 2; do
python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_seg$i.json 2> $o/bench_cfg4_seg.err
VPB_SPLINE_XPLANE=0 python bench.py --config cfg4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg4_twopass$i.json 2> $o/bench_cfg4_twopass.err
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spline_xplane_seg_kernel --launch-skip 2 --launch-count 1 -o $o/splane_seg python scripts/prof_step.py --method spline --dofs 128 128 128 128 --tau 0.1 --steps 5 --advance > $o/ncu.log 2>&1
ncu -i $o/splane_seg.ncu-rep --page raw --csv > $o/splane_seg_raw.csv 2>/dev/null
ls -la $o
