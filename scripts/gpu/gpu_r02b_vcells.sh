# v pass CTA shape: v1 cells per CTA x ring stages (VPB_VCELLS / VPB_VSTAGES
# builds in vlib/) against the default 4 x 4, bench loop at configs 2 and 3
set -x
o=gpurun_out/r02b_vc; mkdir -p $o
for rep in 1 2; do
  python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/def$rep.json 2> $o/def$rep.err
  for v in vc6s4 vc6s3 vc5s4; do
    VPB_LIB=vlib/libvpb200_$v.so python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > $o/${v}_$rep.json 2> $o/${v}_$rep.err
  done
done
python bench.py --config cfg3 --steps 60 --warmup 5 --no-cpu-baseline --no-e2e > $o/c3def.json 2> $o/c3def.err
for v in vc6s4 vc6s3; do
  VPB_LIB=vlib/libvpb200_$v.so python bench.py --config cfg3 --steps 60 --warmup 5 --no-cpu-baseline --no-e2e > $o/c3_$v.json 2> $o/c3_$v.err
done
VPB_LIB=vlib/libvpb200_vc6s4.so timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -m gpu -x -q -p no:cacheprovider -k "vplane or fused_v" > $o/pytest_vc6s4.log 2>&1; echo rc=$? >> $o/pytest_vc6s4.log
ls $o
