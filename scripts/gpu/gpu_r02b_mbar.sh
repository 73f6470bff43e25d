# composed x pass: per-chunk CTA barrier (vlib/libvpb200_bar.so, commit 53b19a6)
# vs mbarrier slot release (in-tree): digests, kernel alone, bench loop, tests
set -x
o=gpurun_out/r02b_mb; mkdir -p $o
python scripts/xcomp_digest.py > $o/digest_mb.json 2>&1
VPB_LIB=vlib/libvpb200_bar.so python scripts/xcomp_digest.py > $o/digest_bar.json 2>&1
VPB_XCOMP_BST=1 python scripts/xcomp_digest.py > $o/digest_mb_bst1.json 2>&1
for rep in 1 2; do
  for c in cfg2 cfg3 cfg5; do
    VPB_LIB=vlib/libvpb200_bar.so python scripts/tune_xcomp.py --config $c --reps 9 | sed "s/^/bar /" >> $o/tune.txt 2>&1
    python scripts/tune_xcomp.py --config $c --reps 9 | sed "s/^/mb /" >> $o/tune.txt 2>&1
  done
  VPB_LIB=vlib/libvpb200_bar.so python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/bench_bar$rep.json 2> $o/bench_bar$rep.err
  python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/bench_mb$rep.json 2> $o/bench_mb$rep.err
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/pytest_gpu.log 2>&1; echo rc=$? >> $o/pytest_gpu.log
ls $o
