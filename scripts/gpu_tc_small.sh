#!/bin/bash
# sweep tile width below the 16-column chunk at small sizes (one wave)
for cfg in "1000 f64" "2000 f64"; do
  for tc in 16 12 10 8 6; do
    DROTB_TC=$tc timeout 300 python scripts/probe_iter.py $cfg 2>&1 | sed "s/\$/ tc=$tc/" | tail -1
  done
done
