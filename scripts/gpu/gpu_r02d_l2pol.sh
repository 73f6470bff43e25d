# fourth session: L2 policy A/B of the composed x pass's density RED.ADDs / streaming copies (configs 5 and 2)
set -x
o=gpurun_out/r02d_l2pol; mkdir -p $o
for v in head rednohint streamnormal head rednohint streamnormal; do
lib=ab/libvpb200_$v.so; [ $v = head ] && lib=paper_1803_02143_b200/libvpb200.so
VPB_LIB=$lib python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $o/bench_cfg5_${v}_$RANDOM.json 2>> $o/err.log
done
for v in head rednohint streamnormal; do
lib=ab/libvpb200_$v.so; [ $v = head ] && lib=paper_1803_02143_b200/libvpb200.so
VPB_LIB=$lib python bench.py --config cfg2 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > $o/bench_cfg2_${v}.json 2>> $o/err.log
done
ls -la $o
