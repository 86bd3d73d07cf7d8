#!/bin/bash
# graph-timed us/iteration
for cfg in "1000 f64" "10000 f32" "2000 f64" "1000 f64"; do
  timeout 300 python scripts/probe_iter.py $cfg 2>&1 | tail -1
done
