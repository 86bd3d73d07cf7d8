#!/bin/bash
# dev aid: build K1 tuning variants of libdrotb200.so (kernels.cu recompiled
# with extra -D flags, every other object from _build/)
# usage: scripts/build_variants.sh NAME "-DFLAG=.. -DFLAG2=.." [NAME2 "FLAGS2" ...]
cd "$(dirname "$0")/../paper_2110_11738_b200" || exit 1
mkdir -p _variants
others=$(ls _build/*.o | grep -v kernels.cu.o)
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -I../include \
      --expt-relaxed-constexpr $flags -c csrc/kernels.cu -o _variants/k_$name.o && \
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/lib_$name.so _variants/k_$name.o \
      $others -lpthread && echo "built $name" ) &
done
wait
