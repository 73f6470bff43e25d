# composed x pass ring depth / chunk / bulk-store plan at config 2:
# kernel alone (tune_xcomp) and in the bench loop
set -x
o=gpurun_out/r02b_st; mkdir -p $o
run() {  # name env...
  name=$1; shift
  for rep in 1 2; do env "$@" python scripts/tune_xcomp.py --config cfg2 --reps 9 | sed "s/^/$name /" >> $o/tune.txt 2>&1; done
  env "$@" python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $o/bench_$name.json 2> $o/bench_$name.err
}
run A VPB_XCOMP_STAGES=3
run B VPB_XCOMP_STAGES=4
run C VPB_XCOMP_STAGES=4 VPB_XCOMP_BST=0
run E VPB_XCOMP_STAGES=5 VPB_XCOMP_BST=0
run F VPB_XCOMP_STAGES=6 VPB_XCOMP_CHUNK=4608 VPB_XCOMP_SMEM=57344
run A2 VPB_XCOMP_STAGES=3
run B2 VPB_XCOMP_STAGES=4
ls $o
