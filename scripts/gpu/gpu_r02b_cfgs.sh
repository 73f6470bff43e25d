# in-bench composed x pass at configs 3 and 5: HEAD of session 1
# (vlib/libvpb200_old.so) vs the running-sum build (in-tree)
set -x
o=gpurun_out/r02b_cfg; mkdir -p $o
for rep in 1 2; do
  VPB_LIB=vlib/libvpb200_old.so python bench.py --config cfg3 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/cfg3_old$rep.json 2> $o/cfg3_old$rep.err
  python bench.py --config cfg3 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/cfg3_new$rep.json 2> $o/cfg3_new$rep.err
done
VPB_LIB=vlib/libvpb200_old.so python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $o/cfg5_old.json 2> $o/cfg5_old.err
python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $o/cfg5_new.json 2> $o/cfg5_new.err
VPB_XCOMP_BST=1 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $o/cfg5_bst1.json 2> $o/cfg5_bst1.err
ls $o
