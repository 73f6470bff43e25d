# v pass with contracted products (build flag VPB_STEP_FMA=1 on fused.cu,
# vlib/libvpb200_vfma.so) vs the reference operation order: bench loop + the
# headline parity tests against the live reference
set -x
o=gpurun_out/r02b_vfma; mkdir -p $o
for rep in 1 2; do
  python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/def$rep.json 2> $o/def$rep.err
  VPB_LIB=vlib/libvpb200_vfma.so python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/vfma$rep.json 2> $o/vfma$rep.err
done
VPB_LIB=vlib/libvpb200_vfma.so timeout 900 python -m pytest tests/test_gpu_parity_headline.py -m gpu -q -p no:cacheprovider -k "config1 or twostream" > $o/pytest_vfma.log 2>&1; echo rc=$? >> $o/pytest_vfma.log
ls $o
