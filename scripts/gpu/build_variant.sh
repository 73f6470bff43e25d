#!/bin/bash
# build ab/libvpb200_<name>.so with extra nvcc flags for the listed sources
# (the other objects come from the in-tree build); load it with VPB_LIB=...
# usage: build_variant.sh NAME "fused fused2 xcomp" -DFOO=1 ...
set -e
cd "$(dirname "$0")/../.."
name=$1; shift
srcs=$1; shift
python -c "import paper_1803_02143_b200._build as b; b.build()"
d=build/var_$name; mkdir -p $d ab
for s in $srcs; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off,-O2 \
    -I include "$@" -c paper_1803_02143_b200/csrc/$s.cu -o $d/$s.o &
done
wait
objs=""
for o in common dg fused fused2 xcomp spline field halo; do
  if [ -f $d/$o.o ]; then objs="$objs $d/$o.o"; else objs="$objs build/obj/$o.o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart=static -o ab/libvpb200_$name.so $objs
echo ab/libvpb200_$name.so
