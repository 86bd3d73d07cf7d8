#!/bin/bash
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
for v in 0 1; do echo "== DROTB_TAIL_PDL=$v"; DROTB_TAIL_PDL=$v timeout 300 python scripts/probe_timeline.py 10000 f32 2>&1 | tail -17; done
for v in 0 1; do echo "== DROTB_TAIL_PDL=$v"; DROTB_TAIL_PDL=$v timeout 300 python scripts/probe_timeline.py 1000 f64 2>&1 | tail -17; done
timeout 900 python -m pytest tests -m gpu -q -x -k "tail or golden_fast or api or sweep or c4_grid_fast" 2>&1 | tail -3
