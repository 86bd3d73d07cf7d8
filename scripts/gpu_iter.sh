#!/bin/bash
# graph-timed us/iteration, A/B: CTA 0's entry-time dry runs on / off
for cfg in "1000 f64" "10000 f32" "2000 f64" "1000 f64" "10000 f32"; do
  timeout 300 python scripts/probe_iter.py $cfg 2>&1 | tail -1
  DROTB_CTAIL_NODRY=1 timeout 300 python scripts/probe_iter.py $cfg 2>&1 | sed 's/$/ nodry/' | tail -1
done
