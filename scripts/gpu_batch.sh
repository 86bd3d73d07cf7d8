#!/bin/bash
# graph batch length: C1 solve wall time and 10k^2 iteration time
for b in 42 96 152 256; do
  echo "DROTB_BATCH=$b"; DROTB_BATCH=$b timeout 300 python scripts/probe_c1.py 2>&1 | head -3 | tail -2
done
for b in 8 12 20; do
  DROTB_BATCH=$b timeout 300 python scripts/probe_iter.py 10000 f32 2>&1 | sed "s/\$/ batch=$b/" | tail -1
done
