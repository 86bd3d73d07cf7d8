#!/bin/bash
# graph-timed us/iteration: 16- vs 8-CTA cluster tail at small sizes
for cfg in "1000 f64" "2000 f64" "1000 f64" "2000 f64"; do
  DROTB_CTAIL=16 timeout 300 python scripts/probe_iter.py $cfg 2>&1 | tail -1
  DROTB_CTAIL=8 timeout 300 python scripts/probe_iter.py $cfg 2>&1 | tail -1
done
