# fourth session: config 5 composed x pass with fewer, larger CTAs (fewer density slabs in L2)
set -x
o=gpurun_out/r02d_cfg5occ; mkdir -p $o
for rep in 1 2; do
for sm in 0 73000 110000; do
if [ $sm = 0 ]; then
python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $o/bench_cfg5_default_$rep.json 2>> $o/err.log
else
VPB_XCOMP_SMEM=$sm VPB_XCOMP_CHUNK=20736 python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $o/bench_cfg5_smem${sm}_$rep.json 2>> $o/err.log
VPB_XCOMP_SMEM=$sm python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $o/bench_cfg5_smem${sm}_chunkdef_$rep.json 2>> $o/err.log
fi
done
done
ls -la $o
