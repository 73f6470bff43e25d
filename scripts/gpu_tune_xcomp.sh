mkdir -p gpurun_out
for cfg in cfg5 cfg3 cfg2; do
for ch in 9216 13824 18432 27648; do for stg in 3 4 6; do
  VPB_XCOMP_CHUNK=$ch VPB_XCOMP_STAGES=$stg VPB_XCOMP_SMEM=114688 timeout 300 python scripts/tune_xcomp.py --config $cfg 2>&1 | tail -1
done; done; done > gpurun_out/tune_xcomp.log 2>&1
cat gpurun_out/tune_xcomp.log
