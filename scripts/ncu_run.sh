#!/bin/bash
# dev aid: launch lists + full captures at one size/dtype
# usage: scripts/ncu_run.sh TAG SIZE DTYPE
TAG=$1; SZ=${2:-10000}; DT=${3:-f32}
# persistent solver kernel (the product path): launch list + full capture of
# launches of 2 iterations (one fold + one skip sweep each)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python scripts/ncu_probe.py $SZ $DT 8 2 > gpurun_out/l_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 2 -c 1 \
    -o gpurun_out/solve_${TAG} python scripts/ncu_probe.py $SZ $DT 6 2 > gpurun_out/p_${TAG}.log 2>&1
# per-launch path (K1 sweep kernel alone)
DROTB_PERSIST=0 ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 2 -c 2 \
    -o gpurun_out/pass_${TAG} python scripts/ncu_probe.py $SZ $DT 6 > gpurun_out/pp_${TAG}.log 2>&1
tail -2 gpurun_out/p_${TAG}.log gpurun_out/pp_${TAG}.log
