#!/bin/bash
# ncu of one steady-state tail launch (after a sweep, caches as the loop left
# them): scripts/gpu_ncu_tail.sh TAG [kernel-regex] [m] [dtype]
TAG=${1:-nt}
KRE=${2:-tail_kernel}
M=${3:-10000}
DT=${4:-f32}
mkdir -p gpurun_out
ncu --set full --clock-control none --cache-control none --import-source on -k regex:${KRE} -s 6 -c 1 \
    -o gpurun_out/tail_${TAG} python scripts/ncu_probe.py ${M} ${DT} 8 > gpurun_out/nt_${TAG}.log 2>&1
tail -3 gpurun_out/nt_${TAG}.log
