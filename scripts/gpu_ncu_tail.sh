#!/bin/bash
TAG=${1:-nt}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 4 -c 1 \
    -o gpurun_out/tail_${TAG} python scripts/ncu_probe.py 10000 f32 8 > gpurun_out/nt_${TAG}.log 2>&1
tail -3 gpurun_out/nt_${TAG}.log
