# config 5 composed x pass plans in the bench loop: default (T2S, G=2, lane
# stores) vs one-cell chunks with output staging (3 / 4 ring stages)
set -x
o=gpurun_out/r02b_c5; mkdir -p $o
for rep in 1 2; do
  python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $o/def$rep.json 2> $o/def$rep.err
  VPB_XCOMP_CHUNK=6912 VPB_XCOMP_BST=1 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $o/g1bst$rep.json 2> $o/g1bst$rep.err
  VPB_XCOMP_CHUNK=6912 VPB_XCOMP_BST=1 VPB_XCOMP_STAGES=4 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $o/g1bst4_$rep.json 2> $o/g1bst4_$rep.err
done
ls $o
