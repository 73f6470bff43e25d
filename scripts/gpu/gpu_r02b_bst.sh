# composed x pass: HEAD build (vlib/libvpb200_old.so) vs running sums (BST=0)
# vs running sums + bulk-store staging (default plan / forced), digests,
# kernel-alone timing, bench, GPU tests of the touched kernels, ncu captures
set -x
o=gpurun_out/r02b_bst; mkdir -p $o
python scripts/xcomp_digest.py > $o/digest_new.json 2>&1
VPB_XCOMP_BST=1 python scripts/xcomp_digest.py > $o/digest_bst1.json 2>&1
VPB_LIB=vlib/libvpb200_old.so python scripts/xcomp_digest.py > $o/digest_old.json 2>&1
for c in cfg2 cfg3 cfg5; do
  for rep in 1 2; do
    VPB_LIB=vlib/libvpb200_old.so python scripts/tune_xcomp.py --config $c --reps 9 | sed "s/^/old /" >> $o/tune.txt 2>&1
    VPB_XCOMP_BST=0 python scripts/tune_xcomp.py --config $c --reps 9 | sed "s/^/rs /" >> $o/tune.txt 2>&1
    python scripts/tune_xcomp.py --config $c --reps 9 | sed "s/^/auto /" >> $o/tune.txt 2>&1
    VPB_XCOMP_BST=1 python scripts/tune_xcomp.py --config $c --reps 9 | sed "s/^/bst1 /" >> $o/tune.txt 2>&1
  done
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $o/bench_auto.json 2> $o/bench_auto.err
VPB_LIB=vlib/libvpb200_old.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $o/bench_old.json 2> $o/bench_old.err
VPB_XCOMP_BST=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $o/bench_rs.json 2> $o/bench_rs.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $o/bench_auto2.json 2> $o/bench_auto2.err
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/pytest_gpu.log 2>&1; echo rc=$? >> $o/pytest_gpu.log
P="python scripts/prof_adv.py --dofs 192 192 192 192 --steps 2"
$P > $o/prof_plain.log 2>&1 && VPB_XCOMP_BST=0 $P > $o/prof_plain_rs.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"xcomp" -c 1 -o $o/prof_auto $P > $o/ncu_auto.log 2>&1 ; \
  VPB_XCOMP_BST=0 ncu --set full --clock-control none --import-source on -k regex:"xcomp" -c 1 -o $o/prof_rs $P > $o/ncu_rs.log 2>&1; echo ncu_rc=$?
ls -la $o
