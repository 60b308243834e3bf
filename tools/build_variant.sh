#!/bin/bash
# Build a variant of libsaim.so for A/B timing (tools/ab.sh): tools/build_variant.sh out.so [-DNAME=VALUE ...]
# (objects under /tmp/saim_objs; every translation unit is recompiled with the given defines)
OUT=$1; shift
D=/tmp/saim_objs/$(basename $OUT .so); mkdir -p $D
SRC=paper_2501_04971_b200/csrc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for f in $SRC/*.cu; do
  nvcc $FL "$@" -c $f -o $D/$(basename $f .cu).o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $OUT $D/*.o -lcudart && echo built $OUT
