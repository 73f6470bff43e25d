#!/bin/bash
# build ab/libvpb200_<name>.so with extra nvcc flags for fused.cu / fused2.cu
# (the other objects come from the in-tree build); usage: build_variant.sh NAME -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
python -c "import paper_1803_02143_b200._build as b; b.build()"
d=build/var_$name; mkdir -p $d ab
for s in fused fused2; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off,-O2 \
    -I include "$@" -c paper_1803_02143_b200/csrc/$s.cu -o $d/$s.o &
done
wait
objs=""
for o in common dg spline field halo; do objs="$objs build/obj/$o.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart=static -o ab/libvpb200_$name.so $objs $d/fused.o $d/fused2.o
echo ab/libvpb200_$name.so
