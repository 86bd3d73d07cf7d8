#!/bin/bash
# dev aid: build K1 tuning variants of libdrotb200.so into paper_2110_11738_b200/_variants
cd "$(dirname "$0")/../paper_2110_11738_b200" || exit 1
mkdir -p _variants
for v in "$@"; do
  set -- $v
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -I../include \
      -DDROTB_PASS_G=$1 -DDROTB_PASS_MINB=$2 -c csrc/kernels.cu -o _variants/k_$1_$2.o && \
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/lib_$1_$2.so _variants/k_$1_$2.o \
      _build/session.cu.o _build/probgen.cpp.o -lpthread ) &
done
wait
