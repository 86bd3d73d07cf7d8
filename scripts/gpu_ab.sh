#!/bin/bash
# same-box A/B of two builds of libdrotb200.so (abtest/lib_old.so, abtest/lib_new.so)
for rep in 1 2; do
  for v in old new; do
    for cfg in "1000 f64" "2000 f64" "5000 f32"; do
      DROTB_LIB=abtest/lib_$v.so timeout 300 python scripts/probe_iter.py $cfg 2>&1 | sed "s/\$/ $v/" | tail -1
    done
  done
done
