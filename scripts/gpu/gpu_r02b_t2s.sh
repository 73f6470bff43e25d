# config 2 composed x pass: default (224 registers, bulk-store staging, 8 warps/SM)
# vs x2 table in shared memory (168 registers, lane stores, 12 warps/SM), bench loop
set -x
o=gpurun_out/r02b_t2s; mkdir -p $o
for rep in 1 2; do
  python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/def$rep.json 2> $o/def$rep.err
  VPB_XCOMP_T2S=1 VPB_XCOMP_BST=0 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/t2s$rep.json 2> $o/t2s$rep.err
  VPB_XCOMP_T2S=1 VPB_XCOMP_BST=0 python scripts/tune_xcomp.py --config cfg2 --reps 9 | sed "s/^/t2s /" >> $o/tune.txt
  python scripts/tune_xcomp.py --config cfg2 --reps 9 | sed "s/^/def /" >> $o/tune.txt
done
ls $o
