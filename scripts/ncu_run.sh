#!/bin/bash
# dev aid: launch list + full capture of the sweep for one size/dtype
# usage: scripts/ncu_run.sh TAG SIZE DTYPE
TAG=$1; SZ=${2:-10000}; DT=${3:-f32}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python scripts/ncu_probe.py $SZ $DT 8 > gpurun_out/l_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 2 -c 2 \
    -o gpurun_out/pass_${TAG} python scripts/ncu_probe.py $SZ $DT 6 > gpurun_out/p_${TAG}.log 2>&1
tail -2 gpurun_out/p_${TAG}.log
