#!/bin/bash
# ncu launch list + full captures of the fold / skip sweep (K1) and of the
# cooperative tail at one size / dtype (the default fast-order path).
# usage: scripts/ncu_run.sh TAG [SIZE] [DTYPE]
TAG=$1; SZ=${2:-10000}; DT=${3:-f32}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python scripts/ncu_probe.py $SZ $DT 8 > gpurun_out/l_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_kernel_async -s 2 -c 2 \
    -o gpurun_out/pass_${TAG} python scripts/ncu_probe.py $SZ $DT 6 > gpurun_out/pp_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 2 -c 1 \
    -o gpurun_out/tail_${TAG} python scripts/ncu_probe.py $SZ $DT 6 > gpurun_out/pt_${TAG}.log 2>&1
for f in l pp pt; do tail -n 2 gpurun_out/${f}_${TAG}.log; done
