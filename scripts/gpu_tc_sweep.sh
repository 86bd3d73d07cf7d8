#!/bin/bash
for tc in 16 32 48 64; do
  echo "tc=$tc $(DROTB_TC=$tc timeout 120 python scripts/probe_timeline.py 10000 f32 2>&1 | grep -E 'graph-timed|parity' | tr '\n' ' ')"
done
for tc in 32 48 64 96; do
  echo "f64 10k tc=$tc $(DROTB_TC=$tc timeout 120 python scripts/probe_timeline.py 10000 f64 2>&1 | grep -E 'graph-timed' | tr '\n' ' ')"
done
