#!/bin/bash
# timeline probes only (+ a 30 us spin between K1 and the tail)
TAG=${1:-t}
mkdir -p gpurun_out
for sz in "10000 f32" "1000 f64"; do
  timeout 300 python scripts/probe_timeline.py $sz >> gpurun_out/timeline_${TAG}.log 2>&1
  DROTB_TAIL_DELAY_US=30 timeout 300 python scripts/probe_timeline.py $sz >> gpurun_out/timeline_${TAG}.log 2>&1
done
cat gpurun_out/timeline_${TAG}.log
