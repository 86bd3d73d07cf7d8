#!/bin/bash
# dev aid: build K1 tuning variants of libdrotb200.so
# usage: scripts/build_variants.sh NAME "-DFLAG=.. -DFLAG2=.." [NAME2 "FLAGS2" ...]
cd "$(dirname "$0")/../paper_2110_11738_b200" || exit 1
mkdir -p _variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -I../include \
      $flags -c csrc/kernels.cu -o _variants/k_$name.o 2>/dev/null && \
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/lib_$name.so _variants/k_$name.o \
      _build/session.cu.o _build/probgen.cpp.o _build/probgen.cu.o -lpthread ) &
done
wait
