# v pass: per-v2-cell CTA barrier (in-tree) vs mbarrier slot release
# (vlib/libvpb200_vmb.so, -DVPB_VPLANE_MBAR=1): bench loop A/B + v-plane tests
set -x
o=gpurun_out/r02b_vmb; mkdir -p $o
VPB_LIB=vlib/libvpb200_vmb.so timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_dist.py -m gpu -x -q -p no:cacheprovider -k "vplane or v2halo or v2peer or fused_v or vshard" > $o/pytest_vmb.log 2>&1; echo rc=$? >> $o/pytest_vmb.log
for rep in 1 2; do
  python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/def$rep.json 2> $o/def$rep.err
  VPB_LIB=vlib/libvpb200_vmb.so python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/vmb$rep.json 2> $o/vmb$rep.err
done
python bench.py --config cfg3 --steps 60 --warmup 5 --no-cpu-baseline --no-e2e > $o/c3def.json 2> $o/c3def.err
VPB_LIB=vlib/libvpb200_vmb.so python bench.py --config cfg3 --steps 60 --warmup 5 --no-cpu-baseline --no-e2e > $o/c3vmb.json 2> $o/c3vmb.err
ls $o
